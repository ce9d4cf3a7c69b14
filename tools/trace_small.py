"""Host/stream timeline of M = 1 partial updates (development aid): RPD_TRACE_HOST marks, and
optionally an ncu launch list of the last update (run under ncu)."""
import os
import sys
os.environ["RPD_TRACE_HOST"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2403_18761_b200 as P
import rpd_workloads as W
if len(sys.argv) > 2:   # a prebuilt library variant
    import paper_2403_18761_b200.rpd as R
    R._lib = None
    R.load_library(sys.argv[2])

M = int(sys.argv[1]) if len(sys.argv) > 1 else 1
ws = W.make_shape_workload(f"C4m{M}", 200_000, 20_000, seed=0, radius_mode="uniform",
                           n_batches=6, batch_m=M, clusters=min(M, 10))
to = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
ctx = P.RPDContext(0, filter_mode="pruned")
ctx.relations(to(ws.verts), to(ws.tets), to(ws.spheres), to(ws.nbr_off), to(ws.nbr_idx))
ctx.clip()
n_prev = ws.N
for (sph, off, idx) in ws.batches:
    ctx.update_partial(to(sph), to(off), to(idx), to(np.arange(n_prev, len(sph), dtype=np.int32)))
    n_prev = len(sph)
torch.cuda.synchronize()
print("ok", ctx.stats()["n_dirty"])
