"""profiles/ncu_traffic.json from an `ncu --set full` capture of `bench.py --profile-only`.

Usage: python tools/ncu_traffic.py <capture.ncu-rep> <workload> [source note]

Kernels are grouped into the query path's three stages (traverse / select / rerank) by name; the
select stage is every dense_* / select_* kernel of ONE query step (the capture's first step, after
the index build's dense_codes kernels). Bytes are DRAM read/write summed over the stage's launches.
A stage absent from the capture keeps its previous entry (marked with the old source).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"


def stage_of(name: str):
    if name.startswith("dense_codes"):
        return None  # index build
    if name.startswith("traverse"):
        return "traverse"
    if name.startswith("dense_") or name.startswith("select_"):
        return "select"
    if name.startswith("rerank") or name.startswith("topk"):
        return "rerank"
    return None


def main():
    rep, workload = sys.argv[1], sys.argv[2]
    note = sys.argv[3] if len(sys.argv) > 3 else ""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base", "--metrics", METRICS],
                         check=True, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    k = h.index("Kernel Name")
    agg = {}
    seen_traverse = 0
    for r in rows[2:]:
        name = r[k].replace("(anonymous namespace)::", "").replace("void ", "")
        name = name.split("::")[-1] if "::" in name.split("(")[0] else name
        st = stage_of(name)
        if st is None:
            continue
        if st == "traverse":
            seen_traverse += 1
            if seen_traverse > 1:
                break  # one query step only
        a = agg.setdefault(st, {"dram_read_bytes": 0, "dram_write_bytes": 0, "duration_ms": 0.0, "launches": 0})
        d = dict(zip(h, r))
        a["dram_read_bytes"] += int(float(d["dram__bytes_read.sum"]))
        a["dram_write_bytes"] += int(float(d["dram__bytes_write.sum"]))
        a["duration_ms"] += float(d["gpu__time_duration.sum"]) * 1e-6
        a["launches"] += 1
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    old = json.load(open(path)) if os.path.exists(path) else {"kernels": {}}
    kernels = {}
    for st in ("traverse", "select", "rerank"):
        if st in agg:
            agg[st]["duration_ms"] = round(agg[st]["duration_ms"], 4)
            kernels[st] = agg[st]
        elif st in old.get("kernels", {}):
            kernels[st] = dict(old["kernels"][st], note="kept from the previous capture: " + old.get("source", "")[:120])
    doc = {"source": f"ncu --set full --clock-control none, {os.path.basename(rep)}: python bench.py --profile-only "
                     f"--no-cpu-baseline --steps 1 --warmup 1 ({workload}); one query step, DRAM bytes summed over "
                     f"each stage's launches. {note}".strip(),
           "workload": workload, "kernels": kernels}
    with open(path, "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main()
