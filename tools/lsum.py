"""Per-kernel totals of an ncu launch list (time + DRAM bytes): python tools/lsum.py launches.csv"""
import csv, sys
from collections import defaultdict
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi, ui, mi = (h.index(c) for c in ("Kernel Name", "Metric Value", "Metric Unit", "Metric Name"))
agg = defaultdict(lambda: [0, 0.0, 0.0])
sc = {"ns": 1e-6, "us": 1e-3, "ms": 1, "s": 1e3, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1}
bs = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
for r in rows[1:]:
    k = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")[-45:]
    if r[mi] == "gpu__time_duration.sum":
        agg[k][0] += 1
        agg[k][1] += float(r[vi].replace(",", "")) * sc[r[ui]]
    else:
        agg[k][2] += float(r[vi].replace(",", "")) * bs.get(r[ui], 1)
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 14]:
    print(f"{v[1]:9.2f} ms {v[0]:5d} {v[2] / 1e9:8.2f} GB {k}")
