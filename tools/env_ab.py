"""A/B of rpd_envelope build variants (development aid): for each `tag:"-DFLAGS"` the library
is rebuilt with the flags and the C3 envelope distance (100 k boundary samples against the
C3 medial mesh) timed; values and primitive ids must equal the first variant's (the culling
and the visiting order never change the result)."""
import importlib
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import rpd_workloads as W

w = W.make_config("C3")
smp_h = W.boundary_samples(w.verts, w.tets, 100_000, seed=5)
ref = None
for spec in sys.argv[1:]:
    tag, flags = spec.split(":", 1)
    import paper_2403_18761_b200._build as B
    import paper_2403_18761_b200.rpd as R
    B = importlib.reload(B)
    B.NVCC_FLAGS += flags.split()
    B.LIB = B.LIB.replace("librpd.so", f"librpd_{tag}.so")
    B.build(force=True)
    R._lib = None
    R.load_library(B.LIB)
    ctx = R.RPDContext(0, filter_mode="pruned")
    ctx.set_euler(w.tets, len(w.verts))
    ctx.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
    ctx.clip()
    mm = ctx.medial_mesh(device=True)
    smp = torch.as_tensor(smp_h).cuda()
    sph = torch.as_tensor(w.spheres).cuda()
    ts = []
    for rep in range(6):
        torch.cuda.synchronize()
        t = time.perf_counter()
        g, p, ne = ctx.envelope(smp, sph, mm["edges"], mm["faces"], device=True)
        torch.cuda.synchronize()
        if rep:
            ts.append((time.perf_counter() - t) * 1e3)
    out = (g.cpu().numpy(), p.cpu().numpy())
    same = "ref" if ref is None else ("SAME" if np.array_equal(ref[0], out[0]) and
                                       np.array_equal(ref[1], out[1]) else "DIFFERENT")
    if ref is None:
        ref = out
    print(f"{tag:10s} envelope C3 100k samples {np.median(ts):8.3f} ms  evals={int(ne)}  {same}",
          flush=True)
    ctx.close()
