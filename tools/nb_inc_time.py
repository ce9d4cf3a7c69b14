"""Development aid: rpd_neighbors_update over the C4 chain (10 batches of 500) and the M = 1 /
M = 10 chains, host-timed per update (device inputs), for the RPD_NB_HEAVY settings given on
the command line ("default" = unset)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2403_18761_b200 as P  # noqa: E402
import rpd_workloads as W  # noqa: E402

P.build()
ctx = P.RPDContext(0, filter_mode="pruned")
chains = {"C4": W.make_config("C4")}
t_, n_, mode_, _, _ = W.CONFIGS["C3"]
for M in (1, 10):
    chains[f"M{M}"] = W.make_shape_workload(f"C4m{M}", t_, n_, seed=0, radius_mode=mode_,
                                            n_batches=6, batch_m=M, clusters=min(M, 10))
for setting in sys.argv[1:] or ["default"]:
    if setting == "default":
        os.environ.pop("RPD_NB_HEAVY", None)
    else:
        os.environ["RPD_NB_HEAVY"] = setting
    for name, w in chains.items():
        box = W.mesh_box(w.verts)
        ts, rows, ts0 = [], [], []
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
                    rows.append(g["n_rows_block"])
                else:
                    ts0.append((time.perf_counter() - t0) * 1e3)
                n_prev = len(sp)
        print(f"RPD_NB_HEAVY={setting:8s} {name}: update median {np.median(ts):.3f} ms "
              f"(min {min(ts):.3f}; first pass {np.median(ts0):.3f}), rows on blocks "
              f"{int(np.median(rows))}", flush=True)
