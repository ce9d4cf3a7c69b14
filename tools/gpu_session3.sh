set -x
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_s3.log 2>&1
python bench.py --config C5 --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python tools/step_once.py C5 pruned 0 > gpurun_out/ncu_c5.log 2>&1
tail -3 gpurun_out/gpu_tests_s3.log; cat gpurun_out/bench_c5.json; tail -5 gpurun_out/bench_c5.err
