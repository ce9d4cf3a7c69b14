#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_graph.py tests/test_gpu_partial.py tests/test_gpu_gather.py tests/test_gpu_parity.py -x -q > gpurun_out/g_tests.log 2>&1
echo "exit $?" >> gpurun_out/g_tests.log
timeout 300 python tools/trace_small_m.py 1 12 > gpurun_out/g_m1.log 2>&1
timeout 600 python bench.py > gpurun_out/g_bench.json 2> gpurun_out/g_bench.err
