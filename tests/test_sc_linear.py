"""SC-Linear on the GPU: suco_gpu_sc_scores / suco_gpu_sc_linear_batch against the
reference's own compute_sc_scores / sc_linear_query (sc_linear.cpp:49-121) run through oracle/_ref,
on the same layout (the GPU index's serialized bytes loaded by the reference)."""
import numpy as np
import pytest


def _pair(gpu, ref, base, params):
    idx = gpu.build_index(base, params)
    return idx, ref.load_index(idx.serialize())


def test_ref_sc_scores_tally(suco, oracle, ref):
    """Host-side sanity of the checker: every subspace hands out exactly c collisions."""
    full = oracle.clustered(600, 12, 6, 3, 0, 50, 6, False)
    ridx = ref.build_index(full, 3, 4, 2, 42)
    q = full[5]
    for alpha in (0.01, 0.1, 1.0):
        sc = ridx.sc_scores(full, q, alpha)
        c = suco.collision_count(alpha, 600)
        assert int(sc.sum()) == 3 * c
        assert sc.max() <= 3


@pytest.mark.gpu
@pytest.mark.parametrize("mode,quant,d,ns", [
    (0, False, 20, 4), (0, True, 20, 4), (1, False, 20, 3), (1, True, 24, 4), (0, False, 7, 3), (1, False, 9, 2),
])
def test_sc_scores_match_reference(gpu, oracle, ref, mode, quant, d, ns):
    full = oracle.clustered(2500 + 8, d, 12, 11 + d, 0, 120, 9, quant)
    base, qs = oracle.hold_out(full, 8, 12)
    idx, ridx = _pair(gpu, ref, base, gpu.IndexParams(ns, 6, 2, 7, gpu.SubspaceMode(mode)))
    for alpha in (0.01, 0.05, 0.3):
        for q in qs[:4]:
            got = idx.sc_scores(q, alpha)
            want = ridx.sc_scores(base, q, alpha)
            assert np.array_equal(got, want), (mode, quant, d, ns, alpha)


@pytest.mark.gpu
@pytest.mark.parametrize("mode,quant,k", [(0, False, 10), (0, True, 10), (1, False, 10), (1, True, 40), (0, False, 1)])
def test_sc_linear_matches_reference(gpu, oracle, ref, mode, quant, k, monkeypatch):
    monkeypatch.setenv("SUCO_SC_BATCH", "5")  # 12 queries: batches of 5, 5 and 2
    full = oracle.clustered(3000 + 12, 24, 15, 40 + k, 0, 200, 12, quant)
    base, qs = oracle.hold_out(full, 12, 41)
    idx, ridx = _pair(gpu, ref, base, gpu.IndexParams(4, 8, 2, 42, gpu.SubspaceMode(mode)))
    for alpha, beta in ((0.05, 0.005), (0.1, 0.02), (0.02, 0.05)):
        ids, dd = idx.sc_linear_batch(qs, gpu.CollisionParams(alpha, beta, k))
        for i, q in enumerate(qs):
            wi, wd = ridx.sc_linear_query(base, q, alpha, beta, k)
            assert np.array_equal(ids[i], wi), (mode, quant, k, alpha, beta, i)
            assert np.array_equal(dd[i], wd), (mode, quant, k, alpha, beta, i)


@pytest.mark.gpu
def test_sc_linear_ties_and_extremes(gpu, ref):
    """Integer data from a tiny range: most distances tie, so the (distance, id) and (score, id) orders
    decide the sets. alpha = beta = 1 makes every point a candidate: the exact kNN."""
    rng = np.random.default_rng(5)
    base = rng.integers(0, 3, size=(300, 8)).astype(np.float32)
    qs = rng.integers(0, 3, size=(5, 8)).astype(np.float32)
    for mode in (0, 1):
        idx, ridx = _pair(gpu, ref, base, gpu.IndexParams(2, 3, 2, 42, gpu.SubspaceMode(mode)))
        for alpha, beta, k in ((0.01, 0.01, 5), (0.5, 0.1, 20), (1.0, 1.0, 300), (1.0, 0.001, 3)):
            ids, dd = idx.sc_linear_batch(qs, gpu.CollisionParams(alpha, beta, k))
            for i, q in enumerate(qs):
                assert np.array_equal(idx.sc_scores(q, alpha), ridx.sc_scores(base, q, alpha))
                wi, wd = ridx.sc_linear_query(base, q, alpha, beta, k)
                assert np.array_equal(ids[i], wi) and np.array_equal(dd[i], wd), (mode, alpha, beta, k, i)
        ti, td = idx.exact_knn_batch(qs, 300)
        ids, dd = idx.sc_linear_batch(qs, gpu.CollisionParams(1.0, 1.0, 300))
        assert np.array_equal(ids, ti) and np.array_equal(dd, td)


@pytest.mark.gpu
def test_sc_linear_errors(gpu):
    """Param validation first (CONFIG, sc_linear.cpp:97), then the query length (CONTRACT)."""
    rng = np.random.default_rng(1)
    base = rng.standard_normal((200, 6)).astype(np.float32)
    idx = gpu.build_index(base, gpu.IndexParams(2, 3, 2, 42))
    q = base[:2]
    with pytest.raises(gpu.ContractError):
        idx.sc_linear_batch(q[:, :5], gpu.CollisionParams(0.1, 0.1, 5))
    with pytest.raises(gpu.ConfigError):
        idx.sc_linear_batch(q[:, :5], gpu.CollisionParams(0.0, 0.1, 5))
    with pytest.raises(gpu.ConfigError):
        idx.sc_linear_batch(q, gpu.CollisionParams(0.1, 1.5, 5))
    with pytest.raises(gpu.ConfigError):
        idx.sc_linear_batch(q, gpu.CollisionParams(0.1, 0.1, 201))
    with pytest.raises(gpu.ContractError):
        idx.sc_scores(q[0, :5], 0.1)
    with pytest.raises(gpu.ConfigError):
        idx.sc_scores(q[0], 1.5)
    ids, dd = idx.sc_linear_batch(np.zeros((0, 6), np.float32), gpu.CollisionParams(0.1, 0.1, 5))
    assert ids.shape == (0, 5)
