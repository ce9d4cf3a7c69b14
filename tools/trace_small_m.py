"""Host/stream timeline of few-insertion partial updates (M = 1 / 10 from the C3 start,
bench.py side_small_m's workload; development aid): RPD_TRACE_HOST marks per update (argument
"trace"; eager path only), and the
per-update device time by CUDA events.  Under ncu, torch fill kernels separate the updates."""
import sys, os
if "trace" in sys.argv[3:]:
    os.environ["RPD_TRACE_HOST"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2403_18761_b200 as P
import rpd_workloads as W
M = int(sys.argv[1]) if len(sys.argv) > 1 else 1
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 6
dev = torch.device("cuda", 0)
to = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(dev)
t_, n_, mode_, _, _ = W.CONFIGS["C3"]
ws = W.make_shape_workload(f"C4m{M}", t_, n_, seed=0, radius_mode=mode_, n_batches=nb,
                           batch_m=M, clusters=min(M, 10))
w3 = W.make_config("C3")
ctx = P.RPDContext(0, filter_mode="pruned")
ctx.relations(to(w3.verts), to(w3.tets), to(ws.spheres), to(ws.nbr_off), to(ws.nbr_idx))
ctx.clip()
n_prev, lat = ws.N, []
marker = torch.empty(1 << 10, device=dev)
for b, (sph, off, idx) in enumerate(ws.batches):
    a = (to(sph), to(off), to(idx), to(np.arange(n_prev, len(sph), dtype=np.int32)))
    n_prev = len(sph)
    torch.cuda.synchronize()
    marker.fill_(float(b))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _, nd = ctx.update_partial(*a)
    e1.record()
    torch.cuda.synchronize()
    lat.append((round(e0.elapsed_time(e1), 4), nd))
print("M", M, "per-update (ms, dirty):", lat, file=sys.stderr)
print("launches per update:", ctx.stats().get("kernel_launches"), file=sys.stderr)
