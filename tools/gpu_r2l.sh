#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2l_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_euler.py -x -q > gpurun_out/r2l_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2l_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-nbr --no-cpu-baseline --no-small > gpurun_out/r2l_bench.json 2> gpurun_out/r2l_bench.err
