# Per-phase cycle shares of the clip kernel (development aid): builds an RPD_CLIP_PHASES
# variant of the library and runs C3 relations + clip a few times.
python - <<'PY'
import sys, os; sys.path.insert(0,'.')
os.environ["RPD_DEBUG_STATS"] = "1"
import paper_2403_18761_b200._build as B
B.NVCC_FLAGS.append("-DRPD_CLIP_PHASES")
B.LIB = B.LIB.replace("librpd.so","librpd_ph.so"); B.build(force=True)
import paper_2403_18761_b200.rpd as R
R._lib=None; R.load_library(B.LIB)
import numpy as np, torch, rpd_workloads as W
w=W.make_config(sys.argv[1] if len(sys.argv) > 1 else "C3")
ctx=R.RPDContext(0, filter_mode="pruned")
args=[torch.as_tensor(np.asarray(a)).cuda() for a in (w.verts,w.tets,w.spheres,w.nbr_off,w.nbr_idx)]
for it in range(3):
    ctx.relations(*args); ctx.clip(); torch.cuda.synchronize()
PY
