#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s_build.log 2>&1
timeout 2400 python tools/ab.py C4 base:"" leaf4:"-DRPD_BVH_LEAF_MINB=4" leaf5:"-DRPD_BVH_LEAF_MINB=5" leaf6:"-DRPD_BVH_LEAF_MINB=6" base2:"" > gpurun_out/s_ab.log 2>&1
