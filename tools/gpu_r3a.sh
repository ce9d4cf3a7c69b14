#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/a_build.log 2>&1
python tools/trace_small_m.py 1 8 > gpurun_out/a_m1.log 2>&1
python tools/trace_small_m.py 10 8 > gpurun_out/a_m10.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/a_m1_launches.csv python tools/trace_small_m.py 1 4 > gpurun_out/a_ncu.log 2>&1
