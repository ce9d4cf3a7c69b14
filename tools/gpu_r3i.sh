#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/i_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_neighbors.py tests/test_gpu_graph.py -x -q > gpurun_out/i_tests.log 2>&1
echo "exit $?" >> gpurun_out/i_tests.log
timeout 900 python bench.py > gpurun_out/i_bench.json 2> gpurun_out/i_bench.err
