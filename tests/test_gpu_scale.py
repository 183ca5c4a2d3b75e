"""Parity at config scale: the BASELINE.json configs' shapes (bench_data.py generators), GPU against
the C oracle on every checked query — ids, distances, candidate sets and per-point SC-scores.

  * cfg1 in full: 100,000 x 128 float rows, all 1,000 queries; the GPU build's `.suco` bytes
    equal the oracle's build of the same rows;
  * cfg2 in full: 1,000,000 x 128 u8-valued rows, all 10,000 queries (the byte re-rank);
  * cfg3 in full: 1,000,000 x 960 float rows, N_s = 16 (two code vectors per point), all 1,000
    queries (the fp32-screened re-rank: d > 128);
  * cfg4's shape at 2,000,000 unit-norm rows (N_s = 8, 64 x 64 cells, alpha = 0.03, beta = 0.005):
    the int8-screened re-rank and the 32-bit dense select at scale;
  * cfg5's shape at 1,000,000 u8 rows (100 x 100 cells: the half-width dense select, a 1 % sampled
    build, alpha = 0.02, beta = 0.002).
"""
import dataclasses
import os
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
sys.path.insert(0, ROOT)


def _cfg(name, **kw):
    import bench_data
    return dataclasses.replace(bench_data.CONFIGS[name], **kw)


def _check(gpu, oracle, idx, oidx, base, qs, cfg, n_inter=3):
    cp = gpu.CollisionParams(cfg.alpha, cfg.beta, cfg.k)
    ids, dd = idx.knn_query_batch(qs, cp)
    oi, od, _ = oidx.knn_query_batch(base, qs, cfg.alpha, cfg.beta, cfg.k)
    bad = np.nonzero(np.any(ids != oi, axis=1) | np.any(dd != od, axis=1))[0]
    assert bad.size == 0, f"{cfg.name}: {bad.size} of {len(qs)} queries differ (first {bad[:5]})"
    for qi in range(n_inter):  # the production select's per-point scores and candidate set
        s1, c1, p1, u1 = idx.query_intermediates(qs[qi], cp)
        s2, c2, p2, u2 = oidx.query_intermediates(base, qs[qi], cfg.alpha, cfg.beta, cfg.k)
        assert np.array_equal(s1, s2), (cfg.name, qi, "scores")
        assert np.array_equal(c1, c2), (cfg.name, qi, "candidates")
        assert np.array_equal(p1, p2) and np.array_equal(u1, u2), (cfg.name, qi, "cells")


def test_cfg1_full_size(gpu, oracle):
    import bench_data
    cfg = _cfg("cfg1")
    base, qs = bench_data.generate(cfg)
    params = gpu.IndexParams(cfg.num_subspaces, cfg.k_half, cfg.iterations, 42)
    idx = gpu.build_index(base, params)
    oidx = oracle.build_index(base, cfg.num_subspaces, cfg.k_half, cfg.iterations, 42, 0)
    assert idx.serialize() == oidx.serialize()
    _check(gpu, oracle, idx, oidx, base, qs, cfg)


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_full_size_all_queries(gpu, oracle, name):
    import bench_data
    cfg = _cfg(name)
    base, qs = bench_data.generate(cfg)
    idx = gpu.build_index(base, gpu.IndexParams(cfg.num_subspaces, cfg.k_half, cfg.iterations, 42))
    oidx = oracle.load_index(idx.serialize())
    _check(gpu, oracle, idx, oidx, base, qs, cfg)


def test_cfg4_shape_2m(gpu, oracle):
    import bench_data
    cfg = _cfg("cfg4", n=2_000_000, queries=2000)
    base, qs = bench_data.generate(cfg)
    idx = gpu.build_index(base, gpu.IndexParams(cfg.num_subspaces, cfg.k_half, cfg.iterations, 42))
    oidx = oracle.load_index(idx.serialize())  # the build's parity is test_cfg1_full_size / test_gpu_build
    _check(gpu, oracle, idx, oidx, base, qs, cfg)


def test_cfg5_shape_half_width_1m(gpu, oracle):
    import bench_data
    cfg = _cfg("cfg5", n=1_000_000, queries=1000)
    base, qs = bench_data.generate(cfg)
    train = bench_data.train_ids(cfg, cfg.n)
    idx = gpu.build_index_sampled(base, train, gpu.IndexParams(cfg.num_subspaces, cfg.k_half, cfg.iterations, 42))
    oidx = oracle.load_index(idx.serialize())
    # the sampled build's centroids are the oracle's k-means on the training rows
    from suco_bytes import parse
    o_train = oracle.build_index(base[train], cfg.num_subspaces, cfg.k_half, cfg.iterations, 42, 0)
    for a, b in zip(parse(idx.serialize())["subspaces"], parse(o_train.serialize())["subspaces"]):
        assert np.array_equal(a["cent1"], b["cent1"]) and np.array_equal(a["cent2"], b["cent2"])
    _check(gpu, oracle, idx, oidx, base, qs, cfg)
