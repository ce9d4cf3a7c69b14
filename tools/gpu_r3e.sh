#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_graph.py -x -q -s > gpurun_out/e_graph.log 2>&1
echo "exit $?" >> gpurun_out/e_graph.log
timeout 600 python bench.py > gpurun_out/e_bench.json 2> gpurun_out/e_bench.err
RPD_GRAPH=0 timeout 600 python bench.py > gpurun_out/e_bench_eager.json 2> gpurun_out/e_bench_eager.err
timeout 600 python bench.py > gpurun_out/e_bench2.json 2> gpurun_out/e_bench2.err
