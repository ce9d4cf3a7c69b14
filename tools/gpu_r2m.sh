#!/bin/bash
# the bench's sharded path (ShardedRPD exchanges, allreduce_euler) through torch.distributed.run
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2m_build.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 bench.py --force-shard --steps 3 --warmup 3 --no-nbr --no-cpu-baseline --no-small > gpurun_out/r2m_bench_shard.json 2> gpurun_out/r2m_bench_shard.err
echo "exit $?" >> gpurun_out/r2m_bench_shard.err
