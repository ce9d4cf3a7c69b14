"""One bench-like step (full RPD + partial updates) for kernel launch lists under ncu."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2403_18761_b200 as P
import rpd_workloads as W
cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
mode = sys.argv[2] if len(sys.argv) > 2 else "pruned"
nb = int(sys.argv[3]) if len(sys.argv) > 3 else 2
w = W.make_config(cfg)
ctx = P.RPDContext(0, filter_mode=mode)
dev = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
base = [dev(w.verts), dev(w.tets), dev(w.spheres), dev(w.nbr_off), dev(w.nbr_idx)]
bat = []
n_prev = w.N
for (s, o, i) in w.batches[:nb]:
    bat.append((dev(s), dev(o), dev(i), dev(np.arange(n_prev, len(s), dtype=np.int32))))
    n_prev = len(s)
for rep in range(2):
    ctx.relations(*base); ctx.clip()
    for b in bat:
        ctx.update_partial(*b)
torch.cuda.synchronize()
print("ok", ctx.stats())
