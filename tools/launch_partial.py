"""Per-kernel times of the last partial update in an ncu launch list."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; data = []
for r in rows:
    if 'Kernel Name' in r: hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get('Metric Name') == 'gpu__time_duration.sum':
            v = float(d['Metric Value'].replace(',', '')); u = d['Metric Unit']
            us = v * {'nsecond': 1e-3, 'usecond': 1.0, 'msecond': 1e3}.get(u, 1.0)
            data.append((d['Kernel Name'].split('(')[0].replace('rpd::', '')[:34], us))
idx = [i for i, (n, _) in enumerate(data) if n == 'k_check_new_ids']
a = idx[-1]
tot = 0
for n, us in data[a:]:
    if n.startswith('k_check_verts') or n.startswith('k_stage_tets'): break
    tot += us; print(f"{us:9.1f}  {n}")
print('partial total us', round(tot, 1))
