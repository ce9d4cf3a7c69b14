# neighbour lists: GPU tests, timing (C3 / C5) and the incremental-update side records
set -u
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/nbh_build.log 2>&1 || { tail gpurun_out/nbh_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_neighbors.py -x -q > gpurun_out/nbh_tests.log 2>&1; echo "tests $?"; tail -3 gpurun_out/nbh_tests.log
timeout 600 python tools/nb_time.py C3 C5 2>&1 | tail -4
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-euler > gpurun_out/nbh_bench.json 2> gpurun_out/nbh_bench.err; echo "bench $?"
python - <<'P'
import json
d = json.loads([l for l in open("gpurun_out/nbh_bench.json") if l.startswith("{")][-1])
print("value", d["value"], "neighbors", d.get("neighbors"))
print("small_m", d.get("partial_small_m"))
P
