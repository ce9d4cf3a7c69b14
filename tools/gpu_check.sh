#!/bin/bash
# One GPU check of the committed state (run under gpurun from the repo root): build, all GPU
# tests, smoke, the default bench line, the C5 bench line and the sharded path through
# torch.distributed.run with one NCCL rank, into gpurun_out/.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/check_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/check_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/check_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/check_smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/check_bench.json 2> gpurun_out/check_bench.err
timeout 1200 python bench.py --config C5 --steps 3 --warmup 3 --no-nbr --no-euler \
    > gpurun_out/check_bench_c5.json 2> gpurun_out/check_bench_c5.err
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 \
    --master-addr=127.0.0.1 --master-port=29531 bench.py --force-shard --steps 3 --warmup 3 \
    --no-nbr --no-euler --no-cpu-baseline > gpurun_out/check_bench_shard.json \
    2> gpurun_out/check_bench_shard.err
