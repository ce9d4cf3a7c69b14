#!/bin/bash
# Round profiling on one B200 (run under gpurun from the repo root):
#   1. the default bench line,
#   2. the per-kernel launch list of one bench step (ncu gpu__time_duration, cold/serialised),
#   3. ncu --set full of the first full-RPD clip launches (fast + wide kernel) and filter kernels
#      of the same bench command.
# Summaries are made here afterwards:  python tools/launch_summary.py gpurun_out/launches_TAG.csv
#                                       python tools/ncu_summary.py gpurun_out/prof_TAG.ncu-rep
set -x
TAG=${1:-r1}
python bench.py --no-nbr > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_${TAG}.log 2>&1
# the dominant kernel (fast clip tier) and the middle tier of the first full RPD
ncu --set full --clock-control none --import-source on -k regex:"k_clip" -c 2 \
    -o gpurun_out/prof_${TAG} python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_full_${TAG}.log 2>&1
# the filter / stage / merge kernels of the first full RPD and first partial update
ncu --set full --clock-control none --import-source on \
    -k regex:"k_bvh_leaf|k_bvh_super|k_bvh_top|k_stage_rows|k_stage_long|k_compact_cands_t|k_compact_pieces|k_rows_update|k_scan|k_pd_" -c 48 \
    -o gpurun_out/prof_${TAG}_aux python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_aux_${TAG}.log 2>&1
tail -c 600 gpurun_out/bench_${TAG}.json
# summaries on the box (the .ncu-rep files are too large to bring back)
python tools/ncu_summary.py gpurun_out/prof_${TAG}.ncu-rep --json gpurun_out/ncu_clip_${TAG}.json > gpurun_out/ncu_clip_${TAG}.txt 2>&1
python tools/ncu_summary.py gpurun_out/prof_${TAG}_aux.ncu-rep --json gpurun_out/ncu_aux_${TAG}.json > gpurun_out/ncu_aux_${TAG}.txt 2>&1
python tools/launch_summary.py gpurun_out/launches_${TAG}.csv > gpurun_out/launch_summary_${TAG}.txt 2>&1
gzip -f gpurun_out/launches_${TAG}.csv
ls -la gpurun_out/*.ncu-rep
rm -f gpurun_out/*.ncu-rep
