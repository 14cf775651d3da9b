"""Summarize an ncu --metrics gpu__time_duration.sum --csv launch list per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr, data = rows[hi], rows[hi + 1:]
ki, vi = hdr.index('Kernel Name'), hdr.index('Metric Value')
agg = collections.defaultdict(lambda: [0, 0.0])
for r in data:
    name = r[ki].split('(')[0][:70]
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(',', ''))
tot = sum(v for c, v in agg.values())
print(f"{'kernel':70s} {'launches':>8s} {'us/launch':>10s} {'share':>6s}")
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:70s} {c:8d} {v / 1e3 / c:10.2f} {100 * v / tot:5.1f}%")
