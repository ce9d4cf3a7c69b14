set -x
TAG=r1e
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_${TAG}.log 2>&1
python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
python bench.py --config C5 --steps 3 --warmup 3 > gpurun_out/bench_c5_${TAG}.json 2> gpurun_out/bench_c5_${TAG}.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-euler --no-small > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-euler --no-small > gpurun_out/ncu_launch_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_clip" -c 2 \
    -o gpurun_out/prof_${TAG} python tools/step_once.py C4 pruned 0 > gpurun_out/ncu_full_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_env_dist" -c 1 \
    -o gpurun_out/prof_${TAG}_env python tools/env_once.py > gpurun_out/ncu_env_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_bvh_leaf|k_bvh_top|k_stage_rows|k_compact_cands_t|k_merge_copy" -c 10 \
    -o gpurun_out/prof_${TAG}_aux python tools/step_once.py C4 pruned 1 > gpurun_out/ncu_aux_${TAG}.log 2>&1
tail -3 gpurun_out/gpu_tests_${TAG}.log
