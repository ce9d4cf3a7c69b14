"""Host/stream timeline of the C4 partial updates (development aid): RPD_TRACE_HOST marks."""
import sys, os
os.environ["RPD_TRACE_HOST"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2403_18761_b200 as P
import rpd_workloads as W
w = W.make_config("C4")
dev = torch.device("cuda", 0)
to = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(dev)
ctx = P.RPDContext(0, filter_mode="pruned")
base = [to(w.verts), to(w.tets), to(w.spheres), to(w.nbr_off), to(w.nbr_idx)]
bat = []
n_prev = w.N
for (s, o, i) in w.batches:
    bat.append((to(s), to(o), to(i), to(np.arange(n_prev, len(s), dtype=np.int32))))
    n_prev = len(s)
for rep in range(3):
    ctx.relations(*base); ctx.clip()
    torch.cuda.synchronize()
    print(f"--- rep {rep}", file=sys.stderr, flush=True)
    for b in bat:
        ctx.update_partial(*b)
