"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv)."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
agg, cnt = defaultdict(float), defaultdict(int)
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(',', ''))
    v *= {'nsecond': 1e-6, 'ns': 1e-6, 'usecond': 1e-3, 'us': 1e-3, 'msecond': 1.0, 'ms': 1.0, 'second': 1e3, 's': 1e3}.get(r[ui].strip(), 1.0)
    name = r[ki].split('(')[0].replace('void ', '').replace('spb::', '')[:50]
    agg[name] += v
    cnt[name] += 1
tot = sum(agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    print("%-50s %5d %10.3f ms %5.1f%%" % (k, cnt[k], v, 100 * v / tot))
print("total %.3f ms" % tot)
