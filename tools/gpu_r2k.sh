#!/bin/bash
# round-2 GPU session C: pool-layout partial updates
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2k_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2k_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2k_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-nbr --no-cpu-baseline > gpurun_out/r2k_bench.json 2> gpurun_out/r2k_bench.err
