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
d = np.concatenate([d, (d[:, 6] >> 32)[:, None]], axis=1)
d[:, 6] &= 0xffffffff
names = ["clk", "rounds", "enum_clk", "scan_clk", "vloop", "n_v", "visits", "start_ns", "visits_grid"]
print("total clk", d[:, 0].sum(), "max", d[:, 0].max(), "enum share", d[:, 2].sum() / d[:, 0].sum(), "scan share", d[:, 3].sum() / d[:, 0].sum())
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
# tail: start / end (ns from the first start) against the radius order
ok = d[:, 7] > 0  # rows written (hidden / empty spheres return early)
t0 = d[ok, 7].min()
d = d.copy()
d[~ok, 7] = t0
st = (d[:, 7] - t0) / 1e6
en = st + d[:, 0] / 1.965e6
print(f"kernel span ~{en.max():.2f} ms; last start {st.max():.2f} ms")
for q in (0.5, 0.9, 0.99):
    print(f"end time p{int(q*100)} {np.quantile(en, q):.2f} ms")
late = np.argsort(-en)[:10]
print("latest finishers: id r start_ms dur_ms")
for i in late:
    print(i, round(float(w.spheres[i][3]), 3), round(st[i], 2), round(d[i, 0] / 1.965e6, 2))
print("r quantiles", np.quantile(w.spheres[:, 3], [0.1, 0.5, 0.9, 1.0]))
# concurrency: spheres in flight over time (a tail of few heavy spheres shows as a low count)
for tq in (0.25, 0.5, 1, 2, 4, 8, 12, 16, 20):
    act = int(((st <= tq) & (en > tq)).sum())
    print(f"t={tq:5.2f} ms: {act} spheres in flight, {int((en <= tq).sum())} done")
print("spheres with dur > 2 ms:", int((d[:, 0] / 1.965e6 > 2).sum()), "> 5 ms:", int((d[:, 0] / 1.965e6 > 5).sum()))
