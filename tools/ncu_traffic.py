"""profiles/ncu_traffic.json: per-stage DRAM bytes of one query step, from ncu evidence.

    python tools/ncu_traffic.py <launches.csv> <cfg> [<full-capture.ncu-rep> <stage> ...]

<launches.csv> is tools/profile_cfg.sh's launch list (gpu__time_duration, dram__bytes_read/write
per launch, one query step of `bench.py --profile-only --steps 1 --warmup 0 --config <cfg>`);
kernels are grouped into the query path's stages (traverse / select / rerank) by name. Each
optional `--set full` capture adds the binding pipes of that stage's top kernel (SM issue, ALU,
LSU / shared wavefronts with the bank-conflict excess, DRAM throughput, occupancy), so bench.py can
say what bounds each stage besides HBM. Entries of other configs are kept.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from launch_table import BYTES, TIME  # noqa: E402

PIPE_METRICS = {
    "issue_busy_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "alu_pct": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "fma_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "fp64_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "lsu_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1_pct": "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smem_ld_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "smem_ld_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "duration_ns": "gpu__time_duration.sum",
}


def stage_of(name: str):
    if name.startswith("dense_codes") or name.startswith("pack_"):
        return None  # index build
    if name.startswith(("traverse", "rank_halves")):
        return "traverse"
    if name.startswith(("dense_", "select_", "shard_")):
        return "select"
    if name.startswith(("rerank", "topk", "merge")):
        return "rerank"
    return None


def clean(name: str) -> str:
    name = name.replace("(anonymous namespace)::", "").replace("void ", "").replace("unnamed>::", "")
    return name.split("(")[0].split("<")[0].strip()


def stages_from_launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ui, ii = (h.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    per = {}
    for r in rows[1:]:
        e = per.setdefault(r[ii], {"name": clean(r[ki])})
        v = float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            e["ms"] = v * TIME[r[ui]]
        else:
            e[r[mi]] = v * BYTES[r[ui]]
    agg = {}
    for e in per.values():
        st = stage_of(e["name"])
        if st is None:
            continue
        a = agg.setdefault(st, {"dram_read_bytes": 0, "dram_write_bytes": 0, "duration_ms": 0.0, "launches": 0,
                                "kernels": {}})
        a["dram_read_bytes"] += int(e.get("dram__bytes_read.sum", 0))
        a["dram_write_bytes"] += int(e.get("dram__bytes_write.sum", 0))
        a["duration_ms"] += e.get("ms", 0.0)
        a["launches"] += 1
        a["kernels"][e["name"]] = round(a["kernels"].get(e["name"], 0.0) + e.get("ms", 0.0), 4)
    for a in agg.values():
        a["duration_ms"] = round(a["duration_ms"], 4)
    return agg


def pipes(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base", "--metrics",
                          ",".join(PIPE_METRICS.values())], check=True, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    best = None
    for r in rows[2:]:
        d = dict(zip(h, r))
        vals = {}
        for k, m in PIPE_METRICS.items():
            try:
                vals[k] = float(d[m].replace(",", ""))
            except (KeyError, ValueError):
                vals[k] = None
        vals["kernel"] = clean(d["Kernel Name"])
        if best is None or (vals["duration_ns"] or 0) > (best["duration_ns"] or 0):
            best = vals
    if best and best.get("smem_ld_wavefronts"):
        w, c = best["smem_ld_wavefronts"], best["smem_ld_conflicts"] or 0.0
        best["smem_ld_excess_x"] = round(w / max(w - c, 1.0), 2)  # wavefronts per conflict-free wavefront
    return best


def main():
    csv_path, cfg = sys.argv[1], sys.argv[2]
    agg = stages_from_launches(csv_path)
    rest = sys.argv[3:]
    for rep, st in zip(rest[0::2], rest[1::2]):
        if st in agg:
            agg[st]["pipes"] = pipes(rep)
            agg[st]["pipes_source"] = os.path.basename(rep)
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    doc = json.load(open(path)) if os.path.exists(path) else {}
    if "workloads" not in doc:
        doc = {"workloads": {}}
    doc["workloads"][cfg] = {
        "source": f"ncu --clock-control none launch list {os.path.basename(csv_path)}: python bench.py --profile-only "
                  f"--no-cpu-baseline --steps 1 --warmup 0 --config {cfg}; one query step, cold caches, serialised "
                  "launches; DRAM bytes summed over each stage's launches",
        "kernels": agg}
    with open(path, "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps(doc["workloads"][cfg], indent=1))


if __name__ == "__main__":
    main()
