import sys; sys.path.insert(0,'.')
import numpy as np, oracle, rpd_workloads as W, paper_2403_18761_b200 as P
from tests.helpers import slice_tets
ctx=P.RPDContext(0)
for seed in range(3):
  for big in (False, True):
    w=W.make_c1(seed, degenerate=True, big=big)
    for wide in (False, True):
        ctx.set_clip_wide(wide)
        ctx.relations(w.verts,w.tets,w.spheres,w.nbr_off,w.nbr_idx); ctx.clip()
        g=ctx.download_cands(); g.update(ctx.download_pieces())
        r=oracle.rpd_workload(w)
        for t in range(w.T):
            a=slice_tets(g,[t]); b=slice_tets(r,[t])
            if not (np.array_equal(a['piece_sphere'],b['piece_sphere']) and np.array_equal(a['piece_facemask'],b['piece_facemask']) and np.array_equal(a['inc_sphere'],b['inc_sphere'])):
                print('seed',seed,'big',big,'wide',wide,'tet',t)
                for x,lab in ((a,'gpu'),(b,'ora')):
                    for p in range(len(x['piece_sphere'])):
                        print(' ',lab, x['piece_sphere'][p], x['piece_facemask'][p], x['inc_sphere'][x['inc_off'][p]:x['inc_off'][p+1]].tolist(), round(x['piece_vol'][p],6))
