"""Development aid: per-source-line warp stall samples of a kernel from an ncu SASS source page
(CSV, --page source --print-source sass) and a local nvdisasm --print-line-info of the same
build (instructions aligned by index, opcodes checked).
    python tools/sass_lines.py page.csv.gz local.sass [top]"""
import collections
import csv
import gzip
import io
import re
import sys

rows = list(csv.reader(io.TextIOWrapper(gzip.open(sys.argv[1]), encoding="utf-8")))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
ins, cur = [], (None, None)
for ln in open(sys.argv[2]).read().splitlines()[1:]:
    if ln.startswith("//---------------------"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;?\s*$", ln)
    if m:
        ins.append((cur, m.group(2)))
assert len(ins) == len(data), (len(ins), len(data))
reasons = ["stall_wait", "stall_long_sb", "stall_short_sb", "stall_branch_resolving",
           "stall_not_selected", "stall_selected", "stall_math", "stall_mio", "stall_lg",
           "stall_barrier", "stall_no_inst", "stall_dispatch"]
agg = collections.defaultdict(lambda: collections.Counter())
tot = collections.Counter()
for (loc, txt), d in zip(ins, data):
    s = int(d["# Samples"] or 0)
    agg[loc]["samples"] += s
    agg[loc]["inst"] += int(d["Instructions Executed"] or 0)
    for r in reasons:
        agg[loc][r] += int(d.get(r) or 0)
    tot["samples"] += s
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
print(f"total samples {tot['samples']}")
for loc, c in sorted(agg.items(), key=lambda kv: -kv[1]["samples"])[:top]:
    st = ", ".join(f"{r[6:]}={c[r]}" for r in sorted(reasons, key=lambda r: -c[r])[:3] if c[r])
    print(f"{100 * c['samples'] / tot['samples']:5.1f}%  {loc[0]}:{loc[1]:<5}  inst {c['inst']:>10}  {st}")
