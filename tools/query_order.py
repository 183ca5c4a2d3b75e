"""Experiment: does the processing order of a batch's queries change the re-rank's DRAM traffic?
Runs one config's batch in the generated order and sorted by the queries' nearest IMI cells of
subspaces 0 and 1 (neighbouring queries share candidates, so concurrent CTAs could share L2 lines)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench_data
import paper_2411_14754_b200 as suco

cfg = bench_data.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg4"]
base, qs = bench_data.generate(cfg)
idx = suco.build_index(base, suco.IndexParams(cfg.num_subspaces, cfg.k_half, cfg.iterations, 42), device=0)
cp = suco.CollisionParams(cfg.alpha, cfg.beta, cfg.k)
dims, sizes, split = idx.layout()
off = [0] + np.cumsum(sizes).astype(int).tolist()
def cell(s):
    c1, c2, _, _ = idx.subspace(s)
    d = dims[off[s]:off[s + 1]]
    h1 = int(split[s])
    x1, x2 = qs[:, d[:h1]], qs[:, d[h1:]]
    a = ((x1[:, None, :] - c1[None]) ** 2).sum(-1).argmin(1)
    b = ((x2[:, None, :] - c2[None]) ** 2).sum(-1).argmin(1)
    return a * cfg.k_half + b
key = cell(0).astype(np.int64) * (cfg.k_half ** 2) + cell(1)
orders = {"generated": np.arange(len(qs)), "by_cells": np.argsort(key, kind="stable"),
          "random": np.random.default_rng(0).permutation(len(qs))}
ctx = idx.context()
ctx.set_profiling(True)
ref = None
for name, o in orders.items():
    q = np.ascontiguousarray(qs[o])
    for it in range(4):
        ids, dd = idx.knn_query_batch(q, cp, scratch=ctx)
        ms, *_ = ctx.stage_times()
    inv = np.empty_like(o); inv[o] = np.arange(len(o))
    ids = ids[inv]
    if ref is None: ref = ids
    print(name, "stage ms (traverse, select, rerank):", np.round(ms, 3), "same:", bool((ids == ref).all()), flush=True)
