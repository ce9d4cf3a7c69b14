#!/bin/bash
# Results table (BASELINE.md layout): one bench line per config, and the C4 headline over seeds
# 0, 1, 2. Writes gpurun_out/res_*.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/res_build.log 2>&1 || exit 1
for c in C2 C3 C5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/res_$c.json 2> gpurun_out/res_$c.err
  echo "$c exit $?"
done
timeout 1500 python tools/seeds.py --config C4 --steps 10 --warmup 3 --out gpurun_out/res_seeds_C4.json > gpurun_out/res_seeds.log 2>&1
echo "seeds exit $?"
