#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/l_build.log 2>&1
timeout 900 python tools/clip_proto/run.py C3 libproto24.so > gpurun_out/l_proto24.log 2>&1
ncu --kernel-name regex:k_proto --launch-count 1 --set full --clock-control none --import-source on -o gpurun_out/l_proto python tools/clip_proto/run.py C3 > gpurun_out/l_ncu.log 2>&1
ncu -i gpurun_out/l_proto.ncu-rep --page details --csv > gpurun_out/l_proto_details.csv 2>&1
rm -f gpurun_out/l_proto.ncu-rep
