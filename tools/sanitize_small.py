"""Small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck / initcheck)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2403_18761_b200 as P
import rpd_workloads as W
for mode in ("all_pairs", "pruned"):
    ctx = P.RPDContext(0, filter_mode=mode)
    for w in (W.make_c1(0), W.make_c1(1, degenerate=True),
              W.make_shape_workload("S", 2000, 150, seed=3, n_batches=2, batch_m=12, clusters=3,
                                    cache=False)):
        for wide in (False, True):
            ctx.set_clip_wide(wide)
            ctx.relations(w.verts, w.tets, w.spheres, w.nbr_off, w.nbr_idx)
            ctx.clip()
            n_old = w.N
            for (s, o, i) in w.batches:
                ctx.update_partial(s, o, i, np.arange(n_old, len(s), dtype=np.int32))
                n_old = len(s)
            ctx.download_pieces()
    ctx.close()
print("sanitize run ok")
