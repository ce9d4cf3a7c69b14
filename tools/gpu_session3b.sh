set -x
TAG=r1c
python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
python tools/euler_once.py C3 > gpurun_out/euler_once.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_clip" -c 1 \
    -o gpurun_out/prof_${TAG}_euler python tools/euler_once.py C3 > gpurun_out/ncu_euler_${TAG}.log 2>&1
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-euler > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-euler > gpurun_out/ncu_launch_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_clip" -c 2 \
    -o gpurun_out/prof_${TAG} python tools/step_once.py C4 pruned 0 > gpurun_out/ncu_full_${TAG}.log 2>&1
tail -c 1500 gpurun_out/bench_${TAG}.json; tail -3 gpurun_out/euler_once.log
