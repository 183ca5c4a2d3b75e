"""Summarise tools/gpu_launch_metrics.sh output: per kernel (first step only) time and DRAM bytes."""
import csv, sys
from collections import OrderedDict
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi, ii = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
d = OrderedDict()
for r in rows[1:]:
    d.setdefault((int(r[ii]), r[ki].split('(')[0][-38:]), {})[r[mi]] = float(r[vi].replace(',', ''))
for (i, k), v in d.items():
    print(f"{i:3d} {k:40s} {v.get('gpu__time_duration.sum', 0) / 1e6:8.3f} ms  rd {v.get('dram__bytes_read.sum', 0) / 1e9:7.3f} GB  wr {v.get('dram__bytes_write.sum', 0) / 1e9:7.3f} GB")
