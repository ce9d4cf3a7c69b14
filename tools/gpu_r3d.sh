#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/d_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_graph.py -x -q -s > gpurun_out/d_graph.log 2>&1
echo "exit $?" >> gpurun_out/d_graph.log
RPD_TRACE_HOST= timeout 300 python tools/trace_small_m.py 1 12 > gpurun_out/d_m1.log 2>&1
timeout 600 python bench.py > gpurun_out/d_bench.json 2> gpurun_out/d_bench.err
RPD_GRAPH=0 timeout 600 python bench.py > gpurun_out/d_bench_eager.json 2> gpurun_out/d_bench_eager.err
timeout 1200 python -m pytest tests/test_gpu_partial.py tests/test_gpu_gather.py tests/test_gpu_euler.py -x -q > gpurun_out/d_partial.log 2>&1
echo "exit $?" >> gpurun_out/d_partial.log
