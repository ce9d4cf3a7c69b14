set -x
TAG=r1d
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_${TAG}.log 2>&1
python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
python bench.py --config C5 --steps 3 --warmup 3 > gpurun_out/bench_c5_${TAG}.json 2> gpurun_out/bench_c5_${TAG}.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5_${TAG}.csv python tools/step_once.py C5 pruned 0 > gpurun_out/ncu_c5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_clip" -c 1 \
    -o gpurun_out/prof_${TAG}_euler python tools/euler_once.py C3 > gpurun_out/ncu_euler_${TAG}.log 2>&1
tail -3 gpurun_out/gpu_tests_${TAG}.log; tail -c 1200 gpurun_out/bench_${TAG}.json
