#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/p_build.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/p_500_warm.csv python tools/trace_small_m.py 500 3 > gpurun_out/p_ncu.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/p_1_warm.csv python tools/trace_small_m.py 1 4 > gpurun_out/p_ncu1.log 2>&1
