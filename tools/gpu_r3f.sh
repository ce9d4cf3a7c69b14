#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/f_build.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/f_m1_warm.csv python tools/trace_small_m.py 1 6 > gpurun_out/f_ncu1.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/f_m500_warm.csv python tools/trace_small_m.py 500 3 > gpurun_out/f_ncu500.log 2>&1
