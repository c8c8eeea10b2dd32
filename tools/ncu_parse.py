"""Summarise an ncu --csv launch/metric list: mean per (kernel, metric)."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]
k, m, v = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value')
acc = defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) <= v:
        continue
    try:
        acc[(r[k].split('(')[0], r[m])].append(float(r[v].replace(',', '')))
    except ValueError:
        pass
for (kn, mn), xs in sorted(acc.items()):
    print(f"{kn[:28]:28s} {mn[:60]:60s} n={len(xs):4d} mean={sum(xs)/len(xs):.4g}")
