# neighbour lists: GPU tests, timing (C3 / C5; line pre-test off / on) and the
# incremental-update side records
set -u
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/nbh_build.log 2>&1 || { tail gpurun_out/nbh_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_neighbors.py -x -q > gpurun_out/nbh_tests.log 2>&1; echo "tests $?"; tail -3 gpurun_out/nbh_tests.log
for lt in 0 1; do echo "RPD_NB_LINE=$lt"; RPD_NB_LINE=$lt timeout 600 python tools/nb_time.py C3 C5 2>&1 | tail -2; done
for h in 2048 32768; do echo "RPD_NB_HEAVY=$h"; RPD_NB_HEAVY=$h timeout 600 python tools/nb_time.py C3 C5 2>&1 | tail -2; done
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-euler > gpurun_out/nbh_bench.json 2> gpurun_out/nbh_bench.err; echo "bench $?"
python - <<'P'
import json
d = json.loads([l for l in open("gpurun_out/nbh_bench.json") if l.startswith("{")][-1])
print("value", d["value"], "neighbors", {k: v for k, v in d.get("neighbors").items() if k != "note"})
print("small_m", d.get("partial_small_m"))
P
