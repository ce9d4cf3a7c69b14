"""Full RPD with the Euler / topology flags: clip time (library events), development aid."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2403_18761_b200 as P
import rpd_workloads as W

w = W.make_config(sys.argv[1] if len(sys.argv) > 1 else "C3")
to = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
base = [to(a) for a in (w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)]
ctx = P.RPDContext(0, filter_mode="pruned")
ctx.set_profile(True)
for eu in (False, True):
    ctx.set_euler(base[1] if eu else None, len(w.verts))
    ts = []
    for r in range(5):
        ctx.relations(*base)
        ctx.clip()
        if r:
            ts.append(ctx.stats()["clip_ms"])
    print("euler" if eu else "plain", f"clip {np.median(ts):.3f} ms")
