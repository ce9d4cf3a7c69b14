#!/bin/bash
# round-2 GPU session B: exchange kernels, bench with breakdown, FP64 peak with clocks
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2b_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_gather.py tests/test_gpu_partial.py -x -q > gpurun_out/r2b_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2b_pytest.log
timeout 120 python tools/fp64_peak.py > gpurun_out/r2b_fp64.log 2>&1
cp profiles/fp64_peak.json gpurun_out/r2b_fp64_peak.json
timeout 900 python bench.py --steps 5 --warmup 3 --no-nbr --no-euler > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
