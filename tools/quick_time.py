"""Quick timing of the RPD path on one config (development aid; bench.py is the contract)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2403_18761_b200 as P
import rpd_workloads as W

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
mode = sys.argv[2] if len(sys.argv) > 2 else "all_pairs"
w = W.make_config(cfg)
print(cfg, W.stats(w), flush=True)
ctx = P.RPDContext(0, filter_mode=mode)
args = [torch.as_tensor(np.asarray(a)).cuda() for a in (w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)]
for it in range(4):
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    torch.cuda.synchronize()
    e0.record(); nc = ctx.relations(*args); e1.record(); c = ctx.clip(); e2.record()
    torch.cuda.synchronize()
    print(f"it{it}: relations {e0.elapsed_time(e1):.3f} ms  clip {e1.elapsed_time(e2):.3f} ms  n_cand {nc} pieces {c.n_pieces} inc {c.n_inc}", flush=True)
print(ctx.stats())
