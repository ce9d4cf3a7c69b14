"""Run tools/fp64_peak (the DFMA microbenchmark, tools/fp64_peak.cu) with nvidia-smi clocks
sampled while it runs; writes profiles/fp64_peak.json (the FP64 roofline denominator of
bench.py) with the clocks it was measured at."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import ClockSampler  # noqa: E402

exe = os.path.join(ROOT, "tools", "fp64_peak")
if not os.path.exists(exe):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", exe,
                           exe + ".cu"])
cs = ClockSampler(0)
cs.start()
out = subprocess.check_output([exe], text=True)
clk = cs.stop()
d = json.loads(out.strip().splitlines()[-1])
d["clocks"] = clk
d["nominal_tflops_at_max_clock"] = round(d["sms"] * 64 * 2 * d["clock_khz_attr"] * 1e3 / 1e12, 3)
with open(os.path.join(ROOT, "profiles", "fp64_peak.json"), "w") as f:
    json.dump(d, f)
print(json.dumps(d))
