#!/bin/bash
# round-2 GPU session D: partial-update timeline (host marks) + per-kernel launch list
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2d_build.log 2>&1
timeout 300 python tools/trace_partial.py > gpurun_out/r2d_trace.log 2>&1
cat > /tmp/one_partial.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2403_18761_b200 as P, rpd_workloads as W
w = W.make_config("C4"); dev = torch.device("cuda", 0)
to = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(dev)
ctx = P.RPDContext(0, filter_mode="pruned")
base = [to(w.verts), to(w.tets), to(w.spheres), to(w.nbr_off), to(w.nbr_idx)]
ctx.relations(*base); ctx.clip()
n_prev = w.N
for (s, o, i) in w.batches[:3]:
    ctx.update_partial(to(s), to(o), to(i), to(np.arange(n_prev, len(s), dtype=np.int32))); n_prev = len(s)
torch.cuda.synchronize()
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2d_launch.csv python /tmp/one_partial.py > gpurun_out/r2d_ncu.log 2>&1
python tools/launch_partial.py gpurun_out/r2d_launch.csv > gpurun_out/r2d_launch_partial.txt 2>&1
