#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b_build.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/b_m1_warm.csv python tools/trace_small_m.py 1 4 > gpurun_out/b_ncu.log 2>&1
RPD_TRACE_HOST= python tools/trace_small_m.py 1 12 > gpurun_out/b_m1_notrace.log 2>&1
