import sys, os, subprocess
sys.path.insert(0, '.')
import numpy as np, rpd_workloads as W
pair = int(sys.argv[1]); seed = int(sys.argv[2])
import paper_2403_18761_b200._build as B
B.NVCC_FLAGS.append(f"-DRPD_TRACE={pair}")
B.LIB = B.LIB.replace("librpd.so", "librpd_trace.so")
B.build(force=True)
import paper_2403_18761_b200.rpd as R
R.load_library(B.LIB)
ctx = R.RPDContext(0)
w = W.make_c1(seed, degenerate=True)
ctx.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
c = ctx.download_cands()
print("pair", pair, "tet", np.searchsorted(c["cand_off"], pair, side="right") - 1, "sphere", c["cand_idx"][pair])
ctx.clip()
import torch; torch.cuda.synchronize()
