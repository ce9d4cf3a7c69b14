"""Run bench.py for workload seeds 0, 1, 2 and report the median (SURVEY.md §8(d) "Seeds 0, 1, 2
per config; report the median").

    python tools/seeds.py [--config C4] [--steps 10] [--warmup 3] [--out FILE] [-- extra bench args]

Each seed is a separate bench.py process (its own workload: mesh jitter, spheres, insertion
batches). The per-seed JSON lines and the medians of the headline keys go to --out.
"""
import argparse
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [("value",), ("e2e", "value"), ("full_rpd_ms",), ("filter_ms",), ("clip_ms",),
        ("partial_rpd_ms",), ("pairs_filtered_per_s",), ("ms_per_step",),
        ("roofline", "frac"), ("partial_small_m", "M1", "partial_ms"),
        ("partial_small_m", "M10", "partial_ms"), ("cpu_baseline", "value")]


def get(d, path):
    for k in path:
        if not isinstance(d, dict) or k not in d:
            return None
        d = d[k]
    return d if isinstance(d, (int, float)) else None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--seeds", default="0,1,2")
    ap.add_argument("--out", default=None)
    ap.add_argument("rest", nargs="*")
    a = ap.parse_args()
    lines = []
    for s in [int(x) for x in a.seeds.split(",")]:
        cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", a.config,
               "--steps", str(a.steps), "--warmup", str(a.warmup), "--seed", str(s)] + a.rest
        out = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT)
        js = [x for x in out.stdout.splitlines() if x.startswith("{")]
        if out.returncode != 0 or not js:
            print(out.stdout[-2000:], out.stderr[-4000:], file=sys.stderr)
            raise SystemExit(f"seed {s}: bench.py failed ({out.returncode})")
        lines.append(json.loads(js[-1]))
        print(f"seed {s}: value {lines[-1]['value']:.4g}", flush=True)
    med = {}
    for path in KEYS:
        v = [get(d, path) for d in lines]
        if all(x is not None for x in v):
            med[".".join(path)] = {"median": float(np.median(v)), "per_seed": v}
    res = {"config": a.config, "seeds": a.seeds, "steps": a.steps, "warmup": a.warmup,
           "median": med, "lines": lines}
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)
    print(json.dumps({"config": a.config, "median": {k: v["median"] for k, v in med.items()}}))


if __name__ == "__main__":
    main()
