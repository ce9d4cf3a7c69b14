"""Kernels of an ncu launch list (gpu__time_duration.sum CSV) between the last two torch fill
kernels (trace_small_m.py's markers): one partial update's launch list."""
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr, rows = rows[0], rows[1:]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
seq = [(r[ki][:64], float(r[vi].replace(",", ""))) for r in rows]
marks = [i for i, (k, _) in enumerate(seq) if "fill" in k.lower()]
which = int(sys.argv[2]) if len(sys.argv) > 2 else -1
a, b = marks[which - 1], marks[which]
tot = 0.0
for k, v in seq[a + 1:b]:
    print(f"{v / 1000:8.2f} us  {k}")
    tot += v
print(f"total {tot / 1000:.2f} us, {b - a - 1} kernels")
