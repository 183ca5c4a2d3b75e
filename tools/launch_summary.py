"""Aggregate an ncu --metrics gpu__time_duration.sum CSV launch list by kernel (times in ms)."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}
agg = collections.OrderedDict()
for r in rows[1:]:
    a = agg.setdefault(r[ki][:70], [0, 0.0])
    a[0] += 1
    a[1] += float(r[vi].replace(",", "")) * scale[r[ui]]
for n, (c, t) in agg.items():
    if t > 0.05:
        print(f"{c:4d} {t:10.3f} ms  ({t / c:8.3f}/launch)  {n}")
