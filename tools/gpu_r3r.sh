#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_graph.py -x -q > gpurun_out/r_tests.log 2>&1
echo "exit $?" >> gpurun_out/r_tests.log
for R in 0 6 10 16; do
  echo "route $R" >> gpurun_out/r_ab.log
  RPD_CLIP_ROUTE=$R timeout 900 python tools/ab.py C4 r$R:@paper_2403_18761_b200/librpd.so >> gpurun_out/r_ab.log 2>&1
done
