#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/q_build.log 2>&1
timeout 1800 python tools/ab.py C4 base:"" rg16:"-DSTAGE_RG=16" minb6:"-DRPD_STAGE_MINB=6" minb8:"-DRPD_STAGE_MINB=8" base2:"" > gpurun_out/q_ab.log 2>&1
