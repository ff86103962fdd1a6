"""Summarise an ncu launch list (gpu__time_duration.sum CSV) per kernel."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
hdr = rows[hi]
ki, vi, ui = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Unit')
agg = defaultdict(lambda: [0, 0.0])
tot = 0.0
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(',', '')) * {'nsecond': 1e-6, 'ns': 1e-6, 'usecond': 1e-3, 'us': 1e-3, 'msecond': 1.0, 'ms': 1.0, 'second': 1e3, 's': 1e3}[r[ui]]
    name = r[ki].split('(')[0]
    agg[name][0] += 1
    agg[name][1] += v
    tot += v
print(f"{'kernel':28s} {'launches':>8s} {'total ms':>10s} {'share':>6s}")
for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:28s} {n:8d} {v:10.3f} {v / tot:6.3f}")
