"""A/B of library variants on partial-update latency for M = 1, 10 and 500 (development aid).
usage: python tools/ab_small.py tag1:"-DFOO=1" tag2:@path/librpd.so ..."""
import importlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import rpd_workloads as W

to = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
sets = {}
for M in (1, 10, 500):
    ws = W.make_config("C4") if M == 500 else W.make_shape_workload(
        f"C4m{M}", 200_000, 20_000, seed=0, radius_mode="uniform", n_batches=6, batch_m=M,
        clusters=min(M, 10))
    base = [to(a) for a in (ws.verts, ws.tets, ws.spheres, ws.nbr_off, ws.nbr_idx)]
    bat, n_prev = [], ws.N
    for (s, o, i) in ws.batches[:6]:
        bat.append((to(s), to(o), to(i), to(np.arange(n_prev, len(s), dtype=np.int32))))
        n_prev = len(s)
    sets[M] = (base, bat)
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
    out = []
    for M, (base, bat) in sets.items():
        ts = []
        for rep in range(3):
            ctx.relations(*base)
            ctx.clip()
            for b in bat:
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                ctx.update_partial(*b)
                e1.record()
                torch.cuda.synchronize()
                if rep > 0:
                    ts.append(e0.elapsed_time(e1))
        out.append(f"M{M} {np.median(ts):.3f}")
    ctx.close()
    print(f"{tag:10s} " + "  ".join(out) + " ms", flush=True)
