#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/h_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_neighbors.py -x -q -s -k incremental > gpurun_out/h_nb.log 2>&1
echo "exit $?" >> gpurun_out/h_nb.log
