"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list (second half = last evaluate)."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h, rows = rows[0], rows[1:]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
part = rows[len(rows) // 2:] if len(sys.argv) < 3 else rows
agg = collections.OrderedDict()
for r in part:
    k = r[ki][:70]
    agg.setdefault(k, [0.0, 0])
    agg[k][0] += float(r[vi].replace(",", "")) / 1000
    agg[k][1] += 1
tot = sum(v[0] for v in agg.values())
for k, v in agg.items():
    print(f"{v[0]:8.1f} us {v[1]:3d}  {k}")
print(f"{tot:8.1f} us total")
