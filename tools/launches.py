"""Summarise an ncu --csv gpu__time_duration launch list per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
data = rows[hi + 1:]
ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
agg = collections.defaultdict(lambda: [0, 0.0, []])
for r in data:
    name = r[ki].split('(')[0][:60]
    v = float(r[vi].replace(',', ''))
    v *= {'nsecond': 1, 'ns': 1, 'usecond': 1e3, 'us': 1e3, 'msecond': 1e6, 'ms': 1e6, 'second': 1e9, 's': 1e9}[r[ui]]
    agg[name][0] += 1
    agg[name][1] += v
    agg[name][2].append(v)
tot = sum(a[1] for a in agg.values())
for k, (n, t, l) in sorted(agg.items(), key=lambda x: -x[1][1]):
    l.sort()
    print(f"{k:60s} n={n:5d} tot={t/1e6:8.2f} ms ({100*t/tot:5.1f}%) med={l[len(l)//2]/1e3:8.1f}us max={l[-1]/1e3:8.1f}us")
print('total ms', tot / 1e6)
