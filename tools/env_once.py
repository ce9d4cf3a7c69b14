"""One envelope-distance call at the bench size (C3 medial mesh, 100k boundary samples)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2403_18761_b200 as P
import rpd_workloads as W

w = W.make_config("C3")
ctx = P.RPDContext(0, filter_mode="pruned")
ctx.set_euler(w.tets, len(w.verts))
ctx.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
ctx.clip()
mm = ctx.medial_mesh(device=True)
smp = torch.as_tensor(W.boundary_samples(w.verts, w.tets, 100_000, seed=5)).cuda()
g, p, ne = ctx.envelope(smp, torch.as_tensor(w.spheres).cuda(), mm["edges"], mm["faces"],
                        device=True)
torch.cuda.synchronize()
print("ok", ne)
