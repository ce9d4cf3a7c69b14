"""A/B of rpd_neighbors build variants (development aid): for each `tag:"-DFLAGS"` the library
is rebuilt with the flags and the C3 (and C5) neighbour lists timed; the lists must be
identical to the first variant's (same algorithm, only rejection order / pruning changes)."""
import importlib
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import rpd_workloads as W

cfgs = [c for c in sys.argv[1].split(",")]
ref = {}
for spec in sys.argv[2:]:
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
    for name in cfgs:
        if name.endswith("inc"):  # the incremental chain of a C4-like workload (C4inc)
            w = W.make_config(name[:-3])
            box = W.mesh_box(w.verts)
            ts = []
            for rep in range(2):
                ctx.neighbors(torch.tensor(w.spheres, device="cuda"), box, device=True)
                n_prev = w.N
                for (sp, _, _) in w.batches:
                    d = torch.tensor(sp, device="cuda")
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    g = ctx.neighbors_update(d, len(sp) - n_prev, box, device=True)
                    torch.cuda.synchronize()
                    if rep:
                        ts.append((time.perf_counter() - t0) * 1e3)
                    n_prev = len(sp)
            print(f"{tag:10s} {name} update median {np.median(ts):8.3f} ms  "
                  f"E={len(g['nbr_idx'])}", flush=True)
            continue
        w = W.make_config(name)
        box = W.mesh_box(w.verts)
        sp = torch.tensor(w.spheres, device="cuda")
        for _ in range(2):
            g = ctx.neighbors(sp, box)
        ts = []
        for _ in range(5):
            torch.cuda.synchronize()
            t = time.perf_counter()
            g = ctx.neighbors(sp, box)
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t) * 1e3)
        key = (name,)
        same = "ref"
        if key not in ref:
            ref[key] = (g["nbr_off"].copy(), g["nbr_idx"].copy())
        else:
            same = "SAME" if (np.array_equal(ref[key][0], g["nbr_off"]) and
                              np.array_equal(ref[key][1], g["nbr_idx"])) else "DIFF"
        print(f"{tag:10s} {name} {np.median(ts):8.2f} ms  E={len(g['nbr_idx'])}  {same}", flush=True)
    ctx.close()
