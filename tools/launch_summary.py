"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel."""
import csv, collections, sys
path = sys.argv[1]
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5   # use the last fraction of launches
rows = list(csv.reader(open(path)))
hdr = None
data = []
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get('Metric Name') == 'gpu__time_duration.sum':
            v = float(d['Metric Value'].replace(',', ''))
            u = d['Metric Unit']
            us = v * {'nsecond': 1e-3, 'ns': 1e-3, 'usecond': 1.0, 'us': 1.0, 'msecond': 1e3, 'ms': 1e3}.get(u, 1.0)
            data.append((d['Kernel Name'].split('(')[0][:48], us))
data = data[int(len(data) * (1 - frac)):]
agg = collections.defaultdict(float); cnt = collections.Counter()
for n, v in data:
    agg[n] += v; cnt[n] += 1
tot = sum(agg.values())
print(f"launches {len(data)}  total {tot:.1f} us")
for n, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"{v:10.1f} us {100*v/tot:5.1f}%  x{cnt[n]:4d}  {n}")
