"""One full RPD with the fractional Euler characteristics (for ncu captures of the EU clip)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2403_18761_b200 as P
import rpd_workloads as W

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
w = W.make_config(cfg)
ctx = P.RPDContext(0, filter_mode="pruned")
dev = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
base = [dev(w.verts), dev(w.tets), dev(w.spheres), dev(w.nbr_off), dev(w.nbr_idx)]
L = ctx.set_euler(base[1], len(w.verts))
ctx.relations(*base)
ctx.clip()
e = ctx.download_euler()
chi = e["rpc_sum"] // L
print("ok L", L, "spheres with cells", int(np.sum(chi != 0)), "euler==1", int(np.sum(chi == 1)))
