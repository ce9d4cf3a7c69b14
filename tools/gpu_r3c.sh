#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_graph.py -x -q -s > gpurun_out/c_graph.log 2>&1
echo "exit $?" >> gpurun_out/c_graph.log
RPD_TRACE_HOST= timeout 300 python tools/trace_small_m.py 1 12 > gpurun_out/c_m1.log 2>&1
RPD_TRACE_HOST= timeout 300 python tools/trace_small_m.py 10 12 > gpurun_out/c_m10.log 2>&1
RPD_GRAPH=0 RPD_TRACE_HOST= timeout 300 python tools/trace_small_m.py 1 12 > gpurun_out/c_m1_eager.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_partial.py tests/test_gpu_gather.py tests/test_gpu_parity.py -x -q > gpurun_out/c_partial.log 2>&1
echo "exit $?" >> gpurun_out/c_partial.log
