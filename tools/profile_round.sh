#!/bin/bash
# Round profiling on one B200 (run under gpurun from the repo root):
#   bench line, per-kernel launch list of one bench step, ncu --set full of the top kernels.
set -x
TAG=${1:-r1}
python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_${TAG}.log 2>&1
python tools/quick_time.py C3 pruned > gpurun_out/qt_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_clip|k_bvh_leaf|k_bvh_super" \
    -s 6 -c 3 -o gpurun_out/prof_${TAG} python tools/quick_time.py C3 pruned \
    > gpurun_out/ncu_full_${TAG}.log 2>&1
tail -c 600 gpurun_out/bench_${TAG}.json
