python - <<'PY'
import sys; sys.path.insert(0,'.')
import paper_2403_18761_b200._build as B
B.NVCC_FLAGS.append("-DRPD_DEBUG_STAGE")
B.LIB = B.LIB.replace("librpd.so","librpd_dbgs.so"); B.build(force=True)
import paper_2403_18761_b200.rpd as R
R.LIB_PATH = B.LIB
R._lib=None; R.load_library(B.LIB)
import numpy as np, torch, rpd_workloads as W
w=W.make_config("C4")
ctx=R.RPDContext(0, filter_mode="pruned")
ctx.relations(w.verts,w.tets,w.spheres,w.nbr_off,w.nbr_idx); ctx.clip(); torch.cuda.synchronize()
print("=== partial", flush=True)
n_old=w.N
for (s,o,i) in w.batches[:1]:
    ctx.update_partial(s,o,i,np.arange(n_old,len(s),dtype=np.int32)); n_old=len(s)
torch.cuda.synchronize()
print("done", ctx.stats())
PY
