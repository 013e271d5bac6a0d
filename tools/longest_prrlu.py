"""Index (among the prrlu_kernel launches of an ncu launch-list CSV) of the longest one: the
--launch-skip value for an `ncu -k regex:prrlu_kernel -c 1` capture of that launch."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, vi = h.index('Kernel Name'), h.index('Metric Value')
d = [float(r[vi].replace(',', '')) for r in rows[hi + 1:] if r[ki].startswith('void <unnamed>::prrlu_kernel<')]
print(max(range(len(d)), key=lambda i: d[i]))
