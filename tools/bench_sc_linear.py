"""SC-Linear on the GPU at a bench config: throughput of suco_gpu_sc_linear_batch,
parity against the reference's sc_linear_query (oracle/_ref) on a few queries, and the quality of
SuCo vs SC-Linear vs the exact kNN (the paper's SC-Linear comparison).

    python tools/bench_sc_linear.py --config cfg2 --queries 200 --ref-queries 3
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench_data  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2", choices=sorted(bench_data.CONFIGS))
    ap.add_argument("--queries", type=int, default=200)
    ap.add_argument("--ref-queries", type=int, default=3)
    args = ap.parse_args()

    import paper_2411_14754_b200 as suco
    from oracle.oracle import ref, ref_available

    cfg = bench_data.CONFIGS[args.config]
    base, queries = bench_data.generate(cfg)
    qs = queries[: args.queries]
    cp = suco.CollisionParams(cfg.alpha, cfg.beta, cfg.k)
    idx = suco.build_index(base, suco.IndexParams(cfg.num_subspaces, cfg.k_half, cfg.iterations, 42))
    idx.sc_linear_batch(qs[:2], cp)  # warm-up (module load)
    t0 = time.perf_counter()
    sl_ids, sl_d = idx.sc_linear_batch(qs, cp)
    gpu_s = time.perf_counter() - t0

    su_ids, su_d = idx.knn_query_batch(qs, cp)
    ti, td = idx.exact_knn_batch(qs, cfg.k)
    out = {
        "workload": cfg.describe(),
        "gpu_sc_linear_qps": len(qs) / gpu_s,
        "gpu_ms_per_query": 1e3 * gpu_s / len(qs),
        "recall_sc_linear": float(np.mean([suco.recall(sl_ids[i], ti[i], cfg.k) for i in range(len(qs))])),
        "recall_suco": float(np.mean([suco.recall(su_ids[i], ti[i], cfg.k) for i in range(len(qs))])),
        "mre_sc_linear": float(np.mean([suco.mre(sl_d[i], td[i], cfg.k) for i in range(len(qs))])),
        "mre_suco": float(np.mean([suco.mre(su_d[i], td[i], cfg.k) for i in range(len(qs))])),
    }
    if ref_available() and args.ref_queries > 0:
        ridx = ref().load_index(idx.serialize())
        same = 0
        t0 = time.perf_counter()
        for i in range(args.ref_queries):
            wi, wd = ridx.sc_linear_query(base, qs[i], cfg.alpha, cfg.beta, cfg.k)
            same += int(np.array_equal(wi, sl_ids[i]) and np.array_equal(wd, sl_d[i]))
        ref_s = time.perf_counter() - t0
        out.update({"ref_sc_linear_qps_1core": args.ref_queries / ref_s, "ref_parity_equal": same,
                    "ref_parity_of": args.ref_queries})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
