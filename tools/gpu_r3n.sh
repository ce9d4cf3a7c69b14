#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/n_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_graph.py tests/test_gpu_partial.py tests/test_gpu_gather.py -x -q > gpurun_out/n_tests.log 2>&1
echo "exit $?" >> gpurun_out/n_tests.log
RPD_GRAPH_TIME=1 timeout 300 python tools/trace_small_m.py 500 6 > gpurun_out/n_500.log 2>&1
RPD_GRAPH_TIME=1 timeout 300 python tools/trace_small_m.py 1 8 > gpurun_out/n_1.log 2>&1
timeout 900 python bench.py > gpurun_out/n_bench.json 2> gpurun_out/n_bench.err
