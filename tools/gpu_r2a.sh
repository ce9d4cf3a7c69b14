#!/bin/bash
# round-2 GPU session A: build, GPU tests, smoke, short bench
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2a_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r2a_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2a_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-nbr > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
