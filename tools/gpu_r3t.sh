#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_gather.py -x -q -k "sphere_volumes" > gpurun_out/t_tests.log 2>&1
echo "exit $?" >> gpurun_out/t_tests.log
