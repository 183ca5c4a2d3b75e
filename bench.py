"""Benchmark: batched SuCo k-NN queries/sec on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl ours|reference]

One step = one pass of the hot path over one batch: all Q queries of the
config (10,000 at cfg2) through centroid distances -> Dynamic Activation ->
SC counting -> top-m select -> exact re-rank -> top-k, with the dataset,
index and queries resident in HBM (`value`), and again end to end through the
C-ABI with pinned host buffers (`e2e`: H2D queries + D2H ids/distances inside
the timed region). Timing: CUDA events on the stream the library launches on,
W untimed warm-up steps, an L2 flush (256 MiB write, outside the events)
between timed steps, max over ranks. Multi-GPU (one process per GPU under
torchrun): cfg1-cfg3 run query-parallel replicas — every rank holds the whole
index (it fits one GPU) and answers its own 10,000-query batch, no data-path
collective, scaling "weak"; cfg4/cfg5 (the configs BASELINE.json shards by
point) and `--sharded` run the library's point-sharded protocol
(suco_gpu_build_shard + suco_gpu_shard_knn_query_batch_device over an NCCL
communicator: each rank generates and holds only its block-cyclic rows, builds
its shard with the k-means jobs spread over the ranks, and answers every query
with three device all-gathers), scaling "strong". `--replicas` forces the
replica mode. `--emulate G` runs G shards on one GPU (in-process communicator,
G host threads) and checks them against the unsharded path.

`--impl reference` times the reference's own CPU implementation
(oracle/_ref/libsuco_ref.so, built from /root/reference sources) on this
host's cores for the same config/metric: each step = a bounded sample of the
queries through run_suco_batch-style knn_query (suco_cli.cpp:95-114).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import bench_data  # noqa: E402


def log(*a):
    print(*a, file=sys.stderr, flush=True)


_JSON_OUT = None


def emit(obj) -> None:
    """The ONE JSON line the driver parses, on the process's original stdout (see main())."""
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(obj) + "\n")
    out.flush()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def ncu_traffic(workload: str) -> dict:
    """Per-stage ncu evidence of one query step of this config (profiles/ncu_traffic.json, written by
    tools/ncu_traffic.py): DRAM bytes (read + write) and, where captured, the binding pipes of the
    stage's top kernel. {} if the config was not profiled."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
    except (OSError, ValueError):
        return {}
    w = t.get("workloads", {}).get(workload)
    if not w:
        return {}
    return {k: {"dram_bytes": v["dram_read_bytes"] + v["dram_write_bytes"], "pipes": v.get("pipes"),
                "ncu_ms": v.get("duration_ms")} for k, v in w["kernels"].items()}


def gather_ceiling(row_bytes: int):
    """GB/s of uniformly random gathers of row_bytes-byte rows on this B200 (profiles/r02_gather_peak.json,
    tools/micro/gather_peak.cu): random row reads cost DRAM per access, so this, not the copy bandwidth,
    is what a re-rank's gathers can reach without locality. None if no matching measurement."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_gather_peak.json")) as f:
            runs = json.load(f)["runs"]
    except (OSError, ValueError, KeyError):
        return None
    for r in runs:
        if r.get("record_bytes") == row_bytes and r.get("read_bytes") == row_bytes:
            return float(r["GBps"])
    return None


def rerank_row_bytes(base, queries, m=None):
    """Bytes the re-rank reads per candidate row: the u8 copy (d padded to 16) for u8-valued data,
    else the int8 screen record (d padded to 16, + 16 bytes of bound terms, padded to 64; from d = 49
    up only its first 64 bytes for most rows) when d % 4 == 0 and d <= 1024 and the candidate lists
    are long enough for the int8 screen (capi.cu upload_data, launch_rerank), else the f32 row."""
    d = base.shape[1]
    u8 = u8_row_bytes(base, queries)
    if u8:
        return u8, "u8 rows"
    if d % 4 == 0 and d <= 1024 and not os.environ.get("SUCO_Q8") == "0" and (m is None or m >= 8192):
        if d > 48:  # the prefix-bound layout (rerank_q8p_kernel, rerank_q8w_kernel for d > 128): the first
            # 64 bytes of every record, the rest for the few rows past the prefix bound
            return 64, "int8 screen record prefixes (+ the rest of the rows past the prefix bound)"
        return ((d + 15) // 16 * 16 + 16 + 63) // 64 * 64, "int8 screen records (+ exact f32 rows of the survivors)"
    return 4 * d, "f32 rows"


def u8_row_bytes(base, queries):
    """Row bytes of the byte re-rank path (d padded to 16) when data and queries are integers in
    [0, 255] and d <= 512 — the library's own certification rule (capi.cu upload_data) — else 0."""
    d = base.shape[1]
    def ok(a):
        return bool(np.all(a == np.trunc(a)) and a.min() >= 0 and a.max() <= 255)
    if d > 512 or os.environ.get("SUCO_NO_U8") or not ok(base) or not ok(queries):
        return 0
    return (d + 15) // 16 * 16


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []  # (arrival time, csv line)
        self.window = None

    def start(self):
        """Start sampling early (before warm-up): nvidia-smi's start-up takes driver locks that
        would otherwise stall the first timed step; summary() keeps the timed window only."""
        self.__enter__()
        time.sleep(1.0)
        return self

    def mark(self):
        self.window = (time.time(), None)

    def stop(self):
        if self.window:
            self.window = (self.window[0], time.time())
        self.__exit__()

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lo, hi = self.window if self.window and self.window[1] else (0.0, float("inf"))
        lines = [ln for t, ln in self.lines if lo <= t <= hi + 0.25] or [ln for _, ln in self.lines[-3:]]
        for ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def run_reference_arm(args, cfg):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle.oracle import ref, ref_available
    if not ref_available():
        emit({"impl": "reference", "unavailable": "oracle/_ref/libsuco_ref.so not built"})
        return
    R = ref()
    base, queries = bench_data.generate(cfg)
    threads = R.hardware_threads()
    t0 = time.time()
    idx = R.build_index(base, cfg.num_subspaces, cfg.k_half, cfg.iterations, 42, 0, 0)
    build_s = time.time() - t0
    sample = args.ref_sample
    rng = np.random.default_rng(7)
    times = []
    for step in range(args.warmup + args.steps):
        sel = np.sort(rng.choice(len(queries), size=min(sample, len(queries)), replace=False))
        _, _, wall = idx.knn_query_batch(base, queries[sel], cfg.alpha, cfg.beta, cfg.k, threads=0)
        if step >= args.warmup:
            times.append(wall)
    qps = sample * len(times) / sum(times)
    line = {
        "impl": "reference", "metric": "batched queries/sec at k=10 (oracle-exact IDs)", "value": qps,
        "unit": "queries/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * sum(times) / len(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded Gaussian mixture, bench_data.py)",
        "config": {"workload": cfg.describe(), "queries_per_step": sample, "build_s": build_s},
        "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": threads, "kind": "reference",
                         "sample": f"{sample} random queries of {cfg.name} per step, run_suco_batch-style "
                                   f"parallel_chunks over {threads} threads; index build {build_s:.1f} s"},
        "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


def main():
    # the driver parses ONE JSON line from stdout: everything else written to file descriptor 1 (NCCL's
    # version banner, native libraries) is sent to stderr, and the JSON line goes to the original stdout
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg4", choices=sorted(bench_data.CONFIGS),
                    help="cfg4 (10M x 96, the largest BASELINE config with an N = 1 point) by default")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--index-source", default="gpu", choices=["gpu", "reference"],
                    help="gpu: suco_gpu_build_index (timed); reference: load the reference CPU build's bytes")
    ap.add_argument("--ref-sample", type=int, default=256, help="queries per step in the reference arm")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU-baseline query time (rank 0)")
    ap.add_argument("--parity-queries", type=int, default=-1,
                    help="queries re-checked against the reference after the timed run (-1: all of them for "
                         "n <= 20M, the CPU-baseline sample otherwise)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-only", action="store_true", help="no L2 flush/e2e/cpu legs (for ncu)")
    ap.add_argument("--no-u8", action="store_true",
                    help="re-rank from the f32 rows even for u8-valued data (the f32-row variant, SURVEY §8(d))")
    ap.add_argument("--sharded", action="store_true", help="use the multi-GPU shard protocol even at N = 1")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: query-parallel full replicas even for the point-sharded configs (cfg4, cfg5)")
    ap.add_argument("--block", type=int, default=0,
                    help="block-cyclic shard block size (ids, a multiple of 2048); 0 = suco_gpu_shard_block_hint")
    ap.add_argument("--emulate", type=int, default=0,
                    help="G > 0: G shards on this one GPU (in-process communicator), checked against the "
                         "unsharded path; per-rank device time reported")
    ap.add_argument("--alpha", type=float, default=None, help="experiment: override the config's alpha")
    ap.add_argument("--beta", type=float, default=None, help="experiment: override the config's beta")
    ap.add_argument("--n", type=int, default=None, help="experiment: override the config's point count")
    ap.add_argument("--queries", type=int, default=None, help="experiment: override the config's query count")
    ap.add_argument("--k", type=int, default=None, help="override the config's k (the reference default is 50)")
    args = ap.parse_args()
    if args.no_u8:
        os.environ["SUCO_NO_U8"] = "1"  # read by the library at index upload
    cfg = bench_data.CONFIGS[args.config]
    if args.alpha is not None or args.beta is not None:
        import dataclasses
        cfg = dataclasses.replace(cfg, alpha=args.alpha if args.alpha is not None else cfg.alpha,
                                  beta=args.beta if args.beta is not None else cfg.beta)
    if args.n is not None or args.queries is not None or args.k is not None:
        import dataclasses
        cfg = dataclasses.replace(cfg, n=args.n or cfg.n, queries=args.queries or cfg.queries, k=args.k or cfg.k)
    sampled = cfg.train_sample < 1.0  # cfg5: centroids trained on a seeded sample (sampled build)

    if args.impl == "reference":
        if sampled:
            emit({"impl": "reference", "unavailable": f"{cfg.name}'s sampled build has no reference "
                              f"API (bench.py --config {cfg.name} reports the reference knn_query on the GPU-built "
                              "index as its cpu_baseline)"})
            return
        run_reference_arm(args, cfg)
        return

    import torch
    import paper_2411_14754_b200 as suco

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    point_sharded = cfg.name in ("cfg4", "cfg5") and not args.replicas  # BASELINE.json: points sharded
    if args.emulate:
        run_emulated(args, cfg)
        return
    if args.sharded or (ws > 1 and point_sharded):
        run_sharded(args, cfg, ws, rank, local)
        return

    t0 = time.time()
    base, queries = bench_data.generate(cfg)
    log(f"[rank {rank}] data {cfg.describe()} generated in {time.time() - t0:.1f}s")
    params = suco.IndexParams(cfg.num_subspaces, cfg.k_half, cfg.iterations, 42, suco.SubspaceMode.Contiguous)
    cp = suco.CollisionParams(cfg.alpha, cfg.beta, cfg.k)
    nq, d, k = len(queries), cfg.d, cfg.k

    ref_idx = None
    ref_build_s = None
    build_s = None
    if args.index_source == "reference":
        from oracle.oracle import ref
        R = ref()
        t0 = time.time()
        ref_idx = R.build_index(base, cfg.num_subspaces, cfg.k_half, cfg.iterations, 42, 0, 0)
        ref_build_s = time.time() - t0
        idx = suco.load_index(ref_idx.serialize(), base, device=local)
    else:
        train = bench_data.train_ids(cfg, len(base)) if sampled else None
        torch.cuda.synchronize()
        t0 = time.time()
        if sampled:
            idx = suco.build_index_sampled(base, train, params, device=local)
        else:
            idx = suco.build_index(base, params, device=local)
        torch.cuda.synchronize()
        build_s = time.time() - t0
    log(f"[rank {rank}] index ready (gpu build {build_s}, reference build {ref_build_s})")

    if ws > 1:  # replicas: each rank answers its own batch (the same set, rotated by rank)
        queries = np.ascontiguousarray(np.roll(queries, rank * (nq // ws), axis=0))
    stream = torch.cuda.Stream()
    ctx = idx.context()  # caller-owned query scratch (query.hpp:72-78)
    dq = torch.from_numpy(queries).cuda()
    dids = torch.empty((nq, k), dtype=torch.int32, device="cuda")
    dd = torch.empty((nq, k), dtype=torch.float64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def step():
        idx.knn_query_batch_device(dq.data_ptr(), nq, d, cp, dids.data_ptr(), dd.data_ptr(), stream.cuda_stream,
                                   scratch=ctx)

    clocks = ClockSampler(local).start()
    for _ in range(args.warmup):
        step()
    stream.synchronize()

    ctx.set_profiling(True)
    step_ms, stage_ms = [], np.zeros(3)
    stats = None
    clocks.mark()
    for _ in range(args.steps):
        if not args.profile_only:
            with torch.cuda.stream(stream):
                flush.fill_(1)
        if ws > 1:
            torch.distributed.barrier()
        stream.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        ms, cum, sq, m = ctx.stage_times()
        stage_ms += ms
        stats = (cum, sq, m)
    clocks.stop()
    ctx.set_profiling(False)
    launches_per_step = ctx.last_launches()  # counted by the library for the last call
    total_ms = sum(step_ms)
    if ws > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    value = ws * nq * args.steps / (total_ms / 1000.0)
    gpu_ids = dids.cpu().numpy().view(np.uint32).copy()
    gpu_d = dd.cpu().numpy().copy()

    # end to end through the C-ABI host entry: pinned host queries in, ids/distances out
    e2e = None
    if not args.profile_only:
        hq = torch.from_numpy(queries).pin_memory()
        hi = torch.empty((nq, k), dtype=torch.int32).pin_memory()
        hd = torch.empty((nq, k), dtype=torch.float64).pin_memory()
        import ctypes as C
        from paper_2411_14754_b200 import _capi
        cpc = cp._c()

        def host_step():
            rc = _capi.knn_query_batch(idx.handle, C.cast(hq.data_ptr(), _capi.f32p), nq, d, C.byref(cpc),
                                       C.cast(hi.data_ptr(), _capi.u32p), C.cast(hd.data_ptr(), _capi.f64p),
                                       ctx.handle)
            if rc:
                raise RuntimeError(_capi.last_error().decode())

        host_step()
        e2e_ms = []
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(1)
            stream.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            host_step()
            e1.record(stream)
            e1.synchronize()
            e2e_ms.append(e0.elapsed_time(e1))
        tot = sum(e2e_ms)
        if ws > 1:
            t = torch.tensor([tot], dtype=torch.float64, device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            tot = float(t.item())
        e2e = {"value": ws * nq * args.steps / (tot / 1000.0), "unit": "queries/s",
               "h2d_bytes_per_step": nq * d * 4, "d2h_bytes_per_step": nq * k * (4 + 8),
               "ms_per_step": tot / args.steps}
        assert np.array_equal(hi.numpy().view(np.uint32), gpu_ids) and np.array_equal(hd.numpy(), gpu_d)

    # answer quality against the GPU exact kNN, on a query sample
    quality = None
    if not args.profile_only and rank == 0:
        sample = min(nq, 1000 if cfg.n <= 20_000_000 else 100)
        t0 = time.time()
        ti, td = idx.exact_knn_batch(queries[:sample], k)
        gt_s = time.time() - t0
        rec = [suco.recall(gpu_ids[i], ti[i], k) for i in range(sample)]
        err = [suco.mre(gpu_d[i], td[i], k) for i in range(sample)]
        quality = {"queries": sample, "recall_at_k": float(np.mean(rec)), "mre": float(np.mean(err)),
                   "ground_truth": "suco_gpu_exact_knn_batch", "ground_truth_s": gt_s}

    # roofline of the dominant stage against the bytes it really moves: the re-rank's rows (u8 /
    # int8-record / f32 bytes per candidate), the select's DRAM bytes measured by ncu (it reads
    # L2-resident point codes, not inverted lists); SURVEY §8(d)'s id-equivalent bytes (u32
    # inverted-list ids + f32 candidate rows) are kept as a labelled secondary figure
    peak, peak_src = measured_peaks()
    cum, sq, m = stats
    stage_avg = stage_ms / args.steps
    row_bytes, row_kind = rerank_row_bytes(base, queries, m)
    traffic = ncu_traffic(cfg.name)
    names = ["traverse", "select", "rerank"]
    id_equiv = {"select": 4.0 * cum, "rerank": 4.0 * d * m * sq + 4.0 * d * sq}
    rr_ncu = (traffic.get("rerank") or {}).get("dram_bytes")
    moved = {"traverse": (traffic.get("traverse") or {}).get("dram_bytes", 0.0),
             "select": (traffic.get("select") or {}).get("dram_bytes"),
             "rerank": rr_ncu or float(row_bytes) * m * sq + 4.0 * d * sq}
    per_kernel = {}
    for i, nm in enumerate(names):
        t = stage_avg[i] / 1000.0
        b = moved[nm]
        per_kernel[nm] = {"ms": stage_avg[i], "moved_bytes": b,
                          "moved_source": "ncu dram bytes" if nm != "rerank" or rr_ncu else f"model: {row_kind}, {row_bytes} B/row",
                          "achieved_gbs": b / t / 1e9 if b else None, "frac": b / t / 1e9 / peak if b else None,
                          "dram_bytes_ncu": (traffic.get(nm) or {}).get("dram_bytes"),
                          "binding_pipes_ncu": (traffic.get(nm) or {}).get("pipes")}
        if nm == "rerank" and b:
            g = gather_ceiling(int(row_bytes))
            if g:  # the re-rank's own ceiling: random row gathers (cost per DRAM access, not per byte)
                per_kernel[nm]["random_gather_ceiling"] = {
                    "gbs": g, "frac": float(row_bytes) * m * sq / t / 1e9 / g,
                    "source": f"profiles/r02_gather_peak.json: uniformly random {int(row_bytes)}-byte rows"}
        if nm in id_equiv:
            per_kernel[nm]["id_equivalent"] = {"bytes": id_equiv[nm], "gbs": id_equiv[nm] / t / 1e9,
                                               "note": "SURVEY 8(d) bytes (u32 ids / f32 rows), not what moves"}
    dom = int(np.argmax(stage_avg))
    dom_name = names[dom]
    dk = per_kernel[dom_name]
    step_s = total_ms / ws / args.steps / 1e3
    path_bytes = sum(v for v in moved.values() if v)
    roofline = {"bound": "hbm", "kernel": dom_name, "achieved": dk["achieved_gbs"], "peak": peak, "unit": "GB/s",
                "frac": dk["frac"], "traffic": dk["dram_bytes_ncu"],
                "traffic_source": "profiles/ncu_traffic.json" if traffic else None, "peak_source": peak_src,
                "binding": dk["binding_pipes_ncu"],
                "query_path": {"bytes_per_step": path_bytes, "achieved": path_bytes / step_s / 1e9,
                               "frac": path_bytes / step_s / 1e9 / peak,
                               "id_equivalent_frac": sum(id_equiv.values()) / step_s / 1e9 / peak},
                "per_kernel": per_kernel}

    # CPU baseline (rank 0, N = 1): the reference itself on a bounded sample of the same queries
    cpu = None
    parity = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline and not args.profile_only:
        try:
            from oracle.oracle import ref, ref_available
            if ref_available():
                R = ref()
                centroids_equal = None
                if ref_idx is None and sampled:
                    # no reference API for the sampled build: the reference's own build_index over the
                    # training rows gives the centroids (they must equal ours), and the reference's
                    # load_index + knn_query run on the GPU-built index bytes
                    sys.path.insert(0, os.path.join(ROOT, "tests"))
                    from suco_bytes import parse
                    t0 = time.time()
                    rs = R.build_index(base[train], cfg.num_subspaces, cfg.k_half, cfg.iterations, 42, 0, 0)
                    ref_build_s = time.time() - t0
                    blob = idx.serialize()
                    a, b = parse(blob), parse(rs.serialize())
                    centroids_equal = all(np.array_equal(x["cent1"], y["cent1"]) and np.array_equal(x["cent2"], y["cent2"])
                                          for x, y in zip(a["subspaces"], b["subspaces"]))
                    del a, b, rs
                    ref_idx = R.load_index(blob)
                    del blob
                elif ref_idx is None:
                    t0 = time.time()
                    ref_idx = R.build_index(base, cfg.num_subspaces, cfg.k_half, cfg.iterations, 42, 0, 0)
                    ref_build_s = time.time() - t0
                threads = R.hardware_threads()
                probe = min(nq, 200 if cfg.n <= 20_000_000 else 16)
                _, _, w = ref_idx.knn_query_batch(base, queries[:probe], cfg.alpha, cfg.beta, k, threads=0)
                sample = int(min(nq, max(probe, args.cpu_seconds * probe / max(w, 1e-6))))
                sel = np.arange(sample)
                ri, rd, wall = ref_idx.knn_query_batch(base, queries[sel], cfg.alpha, cfg.beta, k, threads=0)
                # parity beyond the timed sample: the rest of the batch (untimed), so every query of
                # the step is checked against the reference (--parity-queries bounds it)
                want = args.parity_queries if args.parity_queries >= 0 else (nq if cfg.n <= 20_000_000 else sample)
                want = int(min(nq, max(want, sample)))
                parity_s = wall
                if want > sample:
                    t0 = time.time()
                    ri2, rd2, _ = ref_idx.knn_query_batch(base, queries[sample:want], cfg.alpha, cfg.beta, k,
                                                          threads=0)
                    parity_s += time.time() - t0
                    ri, rd = np.concatenate([ri, ri2]), np.concatenate([rd, rd2])
                    sel = np.arange(want)
                built = (f"reference build_index over the {len(train):,}-row training sample (k-means only) "
                         f"{ref_build_s:.1f} s; queries on the GPU-built index loaded by the reference's load_index"
                         if sampled else f"reference build_index {ref_build_s:.1f} s")
                cpu = {"value": sample / wall, "unit": "queries/s", "cores": threads, "kind": "reference",
                       "sample": f"first {sample} of {nq} {cfg.name} queries through the reference knn_query "
                                 f"(run_suco_batch parallel_chunks, {threads} threads); {built}",
                       "build_s": ref_build_s}
                parity = {"checked_queries": int(len(sel)), "of": nq,
                          "ids_equal": bool(np.array_equal(ri, gpu_ids[sel])),
                          "dists_equal": bool(np.array_equal(rd, gpu_d[sel])),
                          "mismatched_queries": int(np.sum(np.any(ri != gpu_ids[sel], axis=1) |
                                                           np.any(rd != gpu_d[sel], axis=1))),
                          "reference_s": parity_s}
                if sampled:
                    parity["centroids_equal_reference_sample_build"] = centroids_equal
                elif args.index_source == "gpu":
                    parity["index_bytes_equal"] = idx.serialize() == ref_idx.serialize()
        except Exception as e:  # the baseline must not mask the GPU number
            cpu = {"error": repr(e)}

    line = {
        "metric": "batched queries/sec at k=10 (oracle-exact IDs)", "value": value, "unit": "queries/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded Gaussian mixture, bench_data.py; stands in for SIFT1M-shape corpus)",
        "config": {"workload": cfg.describe(), "queries_per_step": nq, "index_build_s": build_s,
                   "index_source": args.index_source, "l2": "256 MiB flush write between timed steps",
                   "rerank_rows": row_kind,
                   "parallelism": f"replicas x{ws}"},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "parity": parity, "quality": quality,
        "gpu_launches": launches_per_step * args.steps, "clocks": clocks.summary(),
    }
    if rank == 0:
        emit(line)
    if ws > 1:
        torch.distributed.destroy_process_group()


def _shard_block(args, cfg, G):
    from paper_2411_14754_b200.sharded import block_hint
    return args.block or block_hint(cfg.n, G)


def run_sharded(args, cfg, ws, rank, local):
    """N GPUs: the library's block-cyclic shard protocol over NCCL. Each rank generates only its own
    rows, builds its shard (k-means jobs spread over the ranks) and answers the whole batch with the
    other ranks (three device all-gathers per tile)."""
    import torch
    import torch.distributed as dist
    import paper_2411_14754_b200 as suco
    from paper_2411_14754_b200.sharded import Comm, Shard

    if not dist.is_initialized():  # --sharded at N = 1 without torchrun
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", local))
    comm = Comm.from_torch(local)
    block = _shard_block(args, cfg, ws)
    t0 = time.time()
    rows, queries = bench_data.generate_shard(cfg, block, ws, rank)
    log(f"[rank {rank}] {len(rows):,} rows of {cfg.describe()} generated in {time.time() - t0:.1f}s (block {block})")
    params = suco.IndexParams(cfg.num_subspaces, cfg.k_half, cfg.iterations, 42, suco.SubspaceMode.Contiguous)
    train = bench_data.train_ids(cfg, cfg.n) if cfg.train_sample < 1.0 else None
    drows = torch.from_numpy(rows).cuda()
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.time()
    shard = Shard.build(drows, cfg.n, params, block, comm, device=local, train_ids=train)
    torch.cuda.synchronize()
    build_s = time.time() - t0
    t = torch.tensor([build_s], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    build_s = float(t.item())
    del drows
    cp = suco.CollisionParams(cfg.alpha, cfg.beta, cfg.k)
    nq, d, k = len(queries), cfg.d, cfg.k
    ctx = shard.context()
    stream = torch.cuda.Stream()
    dq = torch.from_numpy(queries).cuda()
    dids = torch.empty((nq, k), dtype=torch.int32, device="cuda")
    ddist = torch.empty((nq, k), dtype=torch.float64, device="cuda")

    def step():
        shard.knn_query_batch_device(comm, dq.data_ptr(), nq, d, cp, dids.data_ptr(), ddist.data_ptr(),
                                     stream.cuda_stream, scratch=ctx)

    clocks = ClockSampler(local).start()
    for _ in range(args.warmup):
        step()
    stream.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def timed(fn):
        ms = []
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(1)
            stream.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
        t = torch.tensor([sum(ms)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    clocks.mark()
    total_ms = timed(step)
    clocks.stop()
    launches = ctx.last_launches()
    exch = ctx.exchange_bytes()
    hq = torch.from_numpy(queries).pin_memory()
    hi = np.zeros((nq, k), np.uint32)
    hd = np.zeros((nq, k), np.float64)

    def e2e_step():  # host queries in, host results out, through the C-ABI host entry
        import ctypes as C
        from paper_2411_14754_b200 import _capi
        cpc = cp._c()
        with torch.cuda.stream(stream):
            rc = _capi.shard_knn_query_batch(shard.handle, comm.handle, C.cast(hq.data_ptr(), _capi.f32p), nq, d,
                                             C.byref(cpc), hi.ctypes.data_as(_capi.u32p), hd.ctypes.data_as(_capi.f64p),
                                             ctx.handle)
        if rc:
            raise RuntimeError(_capi.last_error().decode())

    e2e_ms = timed(e2e_step)
    consistent = bool(np.array_equal(hi, dids.cpu().numpy().view(np.uint32)) and np.array_equal(hd, ddist.cpu().numpy()))
    value = nq * args.steps / (total_ms / 1000.0)
    peak, peak_src = measured_peaks()
    line = {
        "metric": "batched queries/sec at k=10 (oracle-exact IDs)", "value": value, "unit": "queries/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded Gaussian mixture, bench_data.py; each rank generates only its own rows)",
        "config": {"workload": cfg.describe(), "queries_per_step": nq, "index_build_s": build_s,
                   "parallelism": f"{ws} block-cyclic point shards (block {block}); library shard protocol over "
                                  "NCCL: all-gathers of score totals, block tie counts and local top-k",
                   "exchange_bytes_per_step_per_rank": exch, "l2": "256 MiB flush write between timed steps"},
        "roofline": {"bound": "hbm", "kernel": "whole sharded query path (per-stage times: N = 1 run)",
                     "achieved": None, "peak": peak * ws, "unit": "GB/s", "frac": None, "traffic": None,
                     "peak_source": peak_src},
        "cpu_baseline": None,
        "e2e": {"value": nq * args.steps / (e2e_ms / 1000.0), "unit": "queries/s", "h2d_bytes_per_step": nq * d * 4,
                "d2h_bytes_per_step": nq * k * 12, "ms_per_step": e2e_ms / args.steps},
        "parity": {"host_and_device_entries_agree": consistent,
                   "vs_oracle": "tests/test_sharded.py (G = 1..8 emulated shards, sharded build) and "
                                "bench.py --emulate (full config size)"},
        "gpu_launches": launches * args.steps, "clocks": clocks.summary(),
    }
    if rank == 0:
        emit(line)
    dist.destroy_process_group()


def run_emulated(args, cfg):
    """G shards of the full index on this GPU (in-process communicator on G threads): every rank's
    answer against the unsharded path, the sharded build against cuts of the full build, and each
    rank's device time."""
    import torch
    import paper_2411_14754_b200 as suco
    from paper_2411_14754_b200.sharded import Comm, Shard, run_ranks, shard_ids

    G = args.emulate
    base, queries = bench_data.generate(cfg)
    params = suco.IndexParams(cfg.num_subspaces, cfg.k_half, cfg.iterations, 42, suco.SubspaceMode.Contiguous)
    train = bench_data.train_ids(cfg, cfg.n) if cfg.train_sample < 1.0 else None
    full = suco.build_index_sampled(base, train, params) if train is not None else suco.build_index(base, params)
    cp = suco.CollisionParams(cfg.alpha, cfg.beta, cfg.k)
    want = full.knn_query_batch(queries, cp)
    block = _shard_block(args, cfg, G)
    comms = Comm.local(G)
    t0 = time.time()
    built = run_ranks(lambda r: Shard.build(base[shard_ids(cfg.n, block, G, r)], cfg.n, params, block, comms[r],
                                            train_ids=train), G)
    build_s = time.time() - t0
    same_build = True
    for r in range(G):
        cut = Shard.cut(full, r, G, block)
        for s in range(cfg.num_subspaces):
            a, b = built[r].subspace(s), cut.subspace(s)
            nl = cut.shard_info()["n_local"]
            same_build &= all(np.array_equal(x, y) for x, y in zip(a[:3], b[:3])) and np.array_equal(a[3][:nl], b[3][:nl])
        del cut
    ctxs = [b.context() for b in built]
    outs = run_ranks(lambda r: built[r].knn_query_batch(comms[r], queries, cp, scratch=ctxs[r]), G)
    ok = all(np.array_equal(i, want[0]) and np.array_equal(dd, want[1]) for i, dd in outs)
    # per-rank device time of the protocol with the ranks serialised on one GPU (no overlap)
    dq = torch.from_numpy(queries).cuda()
    outs_d = [(torch.empty((len(queries), cfg.k), dtype=torch.int32, device="cuda"),
               torch.empty((len(queries), cfg.k), dtype=torch.float64, device="cuda")) for _ in range(G)]
    t0 = time.time()
    run_ranks(lambda r: (built[r].knn_query_batch_device(comms[r], dq.data_ptr(), len(queries), cfg.d, cp,
                                                         outs_d[r][0].data_ptr(), outs_d[r][1].data_ptr(),
                                                         scratch=ctxs[r]), ctxs[r].synchronize()), G)
    wall = time.time() - t0
    emit({"emulate": G, "workload": cfg.describe(), "block": block, "sharded_build_equals_cut": same_build,
                      "build_s_emulated": build_s, "ranks_bit_identical_to_unsharded": ok,
                      "exchange_bytes_per_rank": ctxs[0].exchange_bytes(), "wall_s_all_ranks_one_gpu": wall})
    for c in comms:
        c.close()


if __name__ == "__main__":
    main()
