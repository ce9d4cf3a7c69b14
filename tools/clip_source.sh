#!/bin/bash
# Per-source-line stall samples of the fast clip tier (one full-RPD launch at C3), exported
# as CSV (ncu --page source) into gpurun_out/clip_source.csv.gz
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_clip -c 1 \
    -o gpurun_out/clipsrc -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-nbr \
    --no-euler --no-small > gpurun_out/clipsrc.log 2>&1
ncu -i gpurun_out/clipsrc.ncu-rep --page source --csv --print-source cuda > gpurun_out/clip_source.csv 2>&1
ncu -i gpurun_out/clipsrc.ncu-rep --page source --csv --print-source sass > gpurun_out/clip_sass.csv 2>&1
gzip -f gpurun_out/clip_source.csv gpurun_out/clip_sass.csv
rm -f gpurun_out/clipsrc.ncu-rep
ls -la gpurun_out/clip_*
