"""A/B of a clip environment switch (development aid): C3 full RPD + the C4 partial updates,
median clip / step times and a hash of the pieces.  Run once per setting (switches are read
once per process).  Round 2 used it for RPD_CLIP_SORT (pairs in cut-plane-count order; slower,
removed: see DESIGN.md §Clip)."""
import hashlib
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2403_18761_b200 as P
import rpd_workloads as W
w = W.make_config("C4")
dev = torch.device("cuda", 0)
to = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(dev)
ctx = P.RPDContext(0, filter_mode="pruned")
ctx.set_profile(True)
base = [to(w.verts), to(w.tets), to(w.spheres), to(w.nbr_off), to(w.nbr_idx)]
bat, n_prev = [], w.N
for (s, o, i) in w.batches:
    bat.append((to(s), to(o), to(i), to(np.arange(n_prev, len(s), dtype=np.int32))))
    n_prev = len(s)
full, part, steps = [], [], []
for rep in range(8):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    ctx.relations(*base)
    ctx.clip()
    full.append(ctx.stats()["clip_ms"])
    pc = 0.0
    for b in bat:
        ctx.update_partial(*b)
        pc += ctx.stats()["clip_ms"]
    e1.record()
    torch.cuda.synchronize()
    part.append(pc)
    steps.append(e0.elapsed_time(e1))
pcs = ctx.download_pieces()
h = hashlib.sha1(b"".join(np.ascontiguousarray(v).tobytes() for v in pcs.values())).hexdigest()
print(f"{os.environ.get('RPD_CLIP_SORT', '0')}: full clip {np.median(full[2:]):.3f} ms, "
      f"partial clips {np.median(part[2:]):.3f} ms/step, step {np.median(steps[2:]):.3f} ms, "
      f"pieces {h[:12]}", flush=True)
