"""Development aid: per-sphere counters of the neighbour kernel (RPD_NB_DEBUG)."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
os.environ["RPD_NB_DEBUG"] = "gpurun_out/nb_dbg.bin"
import paper_2403_18761_b200 as P  # noqa: E402
import rpd_workloads as W  # noqa: E402

w = W.make_config(sys.argv[1] if len(sys.argv) > 1 else "C3")
ctx = P.RPDContext(0)
g = ctx.neighbors(w.spheres, W.mesh_box(w.verts))
d = np.fromfile("gpurun_out/nb_dbg.bin", dtype=np.int64).reshape(-1, 8)
names = ["clk", "rounds", "enum_clk", "scan", "vloop", "n_v", "n_o", "R_milli"]
print("total clk", d[:, 0].sum(), "max", d[:, 0].max(), "enum share", d[:, 2].sum() / d[:, 0].sum())
for k, n in enumerate(names):
    print(f"{n:8s} mean {d[:, k].mean():12.1f} p50 {np.median(d[:, k]):10.0f} p99 {np.percentile(d[:, k], 99):10.0f} max {d[:, k].max():10d}")
o = np.argsort(-d[:, 0])[:10]
print("top spheres by clk:")
for i in o:
    print(i, w.spheres[i], d[i].tolist(), "rt", w.nbr_off[i + 1] - w.nbr_off[i])
# share of clk by rounds
for r in range(1, 6):
    m = d[:, 1] == r
    print("rounds", r, "spheres", m.sum(), "clk share", d[m, 0].sum() / d[:, 0].sum())
