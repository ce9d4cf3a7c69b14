"""Per-CUDA-source-line instruction/stall summary of an ncu report (source page, cuda,sass)."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
lines = []
fname = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if len(r) > 8 and r[0].isdigit():
        try:
            lines.append((int(r[7] or 0), int(r[4] or 0), fname, int(r[0]), r[1].strip()[:80]))
        except ValueError:
            pass
ti = sum(l[0] for l in lines); ts = sum(l[1] for l in lines)
print(f"total warp-instructions {ti:.3e}  stall samples {ts}")
for l in sorted(lines, reverse=True)[:top]:
    print(f"{100*l[0]/ti:5.1f}% inst {100*l[1]/max(ts,1):5.1f}% stall  {l[2]}:{l[3]}  {l[4]}")
