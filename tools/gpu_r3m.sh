#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m_build.log 2>&1
RPD_GRAPH_TIME=1 timeout 300 python tools/trace_small_m.py 500 6 > gpurun_out/m_500.log 2>&1
RPD_GRAPH_TIME=1 timeout 300 python tools/trace_small_m.py 1 8 > gpurun_out/m_1.log 2>&1
