#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2n_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_gather.py tests/test_gpu_parity.py tests/test_gpu_partial.py -x -q > gpurun_out/r2n_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2n_pytest.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 bench.py --force-shard --steps 3 --warmup 3 --no-nbr --no-cpu-baseline --no-small --no-euler > gpurun_out/r2n_bench_shard.json 2> gpurun_out/r2n_bench_shard.err
