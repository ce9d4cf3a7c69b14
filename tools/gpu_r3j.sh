#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/j_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_cc_sharded.py -x -q > gpurun_out/j_cc.log 2>&1
echo "exit $?" >> gpurun_out/j_cc.log
