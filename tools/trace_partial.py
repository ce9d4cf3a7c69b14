"""Host/stream timeline of the C4 partial updates (development aid): RPD_TRACE_HOST marks."""
import sys, os
os.environ["RPD_TRACE_HOST"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2403_18761_b200 as P
if len(sys.argv) > 1:   # a prebuilt library variant
    import paper_2403_18761_b200.rpd as R
    R._lib = None
    R.load_library(sys.argv[1])
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
import time
tt = []
for rep in range(3):
    ctx.relations(*base); ctx.clip()
    torch.cuda.synchronize()
    print(f"--- rep {rep}", file=sys.stderr, flush=True)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for b in bat:
        ctx.update_partial(*b)
    torch.cuda.synchronize(); tt.append((time.perf_counter() - t0) / len(bat) * 1e3)
print("partial ms (host clock, mean per update) by rep:", [round(x, 3) for x in tt], file=sys.stderr)
st = ctx.stats()
print({k: st[k] for k in ("n_dirty", "pairs_clipped", "n_wide", "max_vertices", "max_planes", "exact_fallbacks", "n_cand", "pairs_tested", "rel_tests")}, file=sys.stderr)
