"""A/B of library variants on the envelope distance at the bench size (development aid)."""
import importlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import rpd_workloads as W

w = W.make_config("C3")
smp = torch.as_tensor(W.boundary_samples(w.verts, w.tets, 100_000, seed=5)).cuda()
sp = torch.as_tensor(w.spheres).cuda()
mm = None
for spec in sys.argv[1:]:
    tag, flags = spec.split(":", 1)
    import paper_2403_18761_b200._build as B
    import paper_2403_18761_b200.rpd as R
    B = importlib.reload(B)
    if flags.startswith("@"):
        B.LIB = flags[1:]
    else:
        B.NVCC_FLAGS += flags.split()
        B.LIB = B.LIB.replace("librpd.so", f"librpd_{tag}.so")
        B.build(force=True)
    R._lib = None
    R.load_library(B.LIB)
    import paper_2403_18761_b200 as P
    ctx = P.RPDContext(0, filter_mode="pruned")
    if mm is None:
        ctx.set_euler(w.tets, len(w.verts))
        ctx.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
        ctx.clip()
        mm = {k: v.clone() for k, v in ctx.medial_mesh(device=True).items()}
    ts = []
    for r in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g, p, ne = ctx.envelope(smp, sp, mm["edges"], mm["faces"], device=True)
        e1.record()
        torch.cuda.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    if tag == sys.argv[1].split(":")[0]:
        g_ref = g.clone()
    print(f"{tag:10s} {np.median(ts):.2f} ms evals {ne} maxdiff {float((g - g_ref).abs().max()):.2e}",
          flush=True)
    ctx.close()
