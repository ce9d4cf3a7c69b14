import sys, numpy as np, torch, os
sys.path.insert(0, ".")
import paper_2403_18761_b200 as P, rpd_workloads as W
w = W.make_config("C4"); dev = torch.device("cuda", 0)
to = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(dev)
ctx = P.RPDContext(0, filter_mode="pruned")
base = [to(a) for a in (w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)]
bat, n_prev = [], w.N
for (s, o, i) in w.batches:
    bat.append((to(s), to(o), to(i), to(np.arange(n_prev, len(s), dtype=np.int32)))); n_prev = len(s)
ts = []
for rep in range(4):
    ctx.relations(*base); ctx.clip()
    for b in bat:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record(); ctx.update_partial(*b); e1.record(); torch.cuda.synchronize()
        if rep >= 2: ts.append(e0.elapsed_time(e1))
st = ctx.stats()
print("partial median %.4f" % np.median(ts), {k: st[k] for k in st if k.startswith("graph")})
