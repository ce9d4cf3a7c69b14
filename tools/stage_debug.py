"""Development aid: per-row cycle report of k_stage_rows (RPD_DEBUG_STAGE build variant) during
the C4 partial updates (rows taking > 100k cycles are printed by the kernel)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2403_18761_b200._build as B
B.NVCC_FLAGS.append("-DRPD_DEBUG_STAGE")
B.NVCC_FLAGS.append("-DRPD_DEBUG_STAGE_MIN=" + os.environ.get("STAGE_MIN", "100000"))
B.LIB = B.LIB.replace("librpd.so", "librpd_dbgstage.so")
B.build(force=True)
import paper_2403_18761_b200.rpd as R
R._lib = None
R.load_library(B.LIB)
import rpd_workloads as W
w = W.make_config("C4")
dev = torch.device("cuda", 0)
to = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(dev)
ctx = R.RPDContext(0, filter_mode="pruned")
ctx.relations(to(w.verts), to(w.tets), to(w.spheres), to(w.nbr_off), to(w.nbr_idx))
ctx.clip()
torch.cuda.synchronize()
print("---- partial updates", flush=True)
n_prev = w.N
for (s, o, i) in w.batches[:2]:
    ctx.update_partial(to(s), to(o), to(i), to(np.arange(n_prev, len(s), dtype=np.int32)))
    n_prev = len(s)
    torch.cuda.synchronize()
    print("---- next", flush=True)
