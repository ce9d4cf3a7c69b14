mkdir -p gpurun_out/r1g
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r1g/gpu_tests_r1g.log 2>&1; echo "rc=$?" >> gpurun_out/r1g/gpu_tests_r1g.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r1g/smoke_r1g.log 2>&1
timeout 900 python bench.py > gpurun_out/r1g/bench_r1g.json 2> gpurun_out/r1g/bench_r1g.err
timeout 300 python tools/nb_time.py > gpurun_out/r1g/nb_time.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_nb --csv --log-file gpurun_out/r1g/ncu_nb_launch.csv python tools/nb_time.py C3 > gpurun_out/r1g/ncu_nb.log 2>&1
tail -2 gpurun_out/r1g/gpu_tests_r1g.log; cat gpurun_out/r1g/smoke_r1g.log | tail -1; tail -c 400 gpurun_out/r1g/bench_r1g.json
