"""Per-kernel table of an ncu launch list (gpu__time_duration + DRAM bytes CSV): launches, total
ms, share of the step, DRAM GB and GB/s.  python tools/launch_table.py <launches.csv>"""
import collections
import csv
import sys

TIME = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}
BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def table(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        a = agg.setdefault(r[ki].split("(")[0][:60], collections.defaultdict(float))
        v = float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            a["ms"] += v * TIME[r[ui]]
            a["n"] += 1
        else:
            a["bytes"] += v * BYTES[r[ui]]
    return agg


if __name__ == "__main__":
    agg = table(sys.argv[1])
    tot = sum(a["ms"] for a in agg.values())
    print(f"{'n':>4} {'ms':>9} {'share':>6} {'DRAM GB':>8} {'GB/s':>8}  kernel")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["ms"]):
        gbs = a["bytes"] / 1e9 / (a["ms"] / 1e3) if a["ms"] else 0.0
        print(f"{int(a['n']):4d} {a['ms']:9.3f} {100 * a['ms'] / tot:5.1f}% {a['bytes'] / 1e9:8.3f} {gbs:8.1f}  {k}")
    print(f"total {tot:.3f} ms")
