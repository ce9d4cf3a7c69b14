#!/bin/bash
# round-2 final-state check: all GPU tests, smoke, default bench, C5 bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2q_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/r2q_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2q_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2q_smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/r2q_bench.json 2> gpurun_out/r2q_bench.err
timeout 1200 python bench.py --config C5 --steps 3 --warmup 3 --no-nbr --no-euler > gpurun_out/r2q_bench_c5.json 2> gpurun_out/r2q_bench_c5.err
