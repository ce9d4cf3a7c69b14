"""Per-CUDA-source-line hot spots of one kernel in an ncu report (warp-stall samples and
executed warp instructions), from `ncu -i REP --page source --csv --print-source cuda,sass`.

usage: python tools/ncu_lines.py REPORT.ncu-rep [launch_index] [top]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
li = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-skip", str(li), "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
fname = ""
lines = []
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) >= 8 and r[0].isdigit() and r[2] == "-":
        samp = int(r[4] or 0)
        inst = int(r[7] or 0)
        lines.append((samp, inst, fname, int(r[0]), r[1].strip()[:90]))
ts = sum(x[0] for x in lines) or 1
ti = sum(x[1] for x in lines) or 1
print(f"samples {ts}  warp-instructions {ti}")
for s, i, f, n, src in sorted(lines, reverse=True)[:top]:
    print(f"{100*s/ts:5.1f}% smp {100*i/ti:5.1f}% ins  {f}:{n:<5d} {src}")
