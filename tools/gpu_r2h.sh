#!/bin/bash
# round-2 GPU session H: slow path parity, compute-sanitizer logs
mkdir -p gpurun_out/sanitizer
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2h_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partial.py -x -q > gpurun_out/r2h_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2h_pytest.log
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_small.py > gpurun_out/sanitizer/$tool.log 2>&1
  echo "exit $?" >> gpurun_out/sanitizer/$tool.log
done
