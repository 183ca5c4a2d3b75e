"""Evaluation: GPU exact kNN against the reference's exact_knn, and recall / mre
against the reference's own known answers (test_eval.cpp:53-82)."""
import math

import numpy as np
import pytest


def test_recall_known_answers(suco):  # test_eval.cpp:53-65
    truth = [3, 7, 9, 1]
    assert suco.recall([3, 7, 9, 1], truth, 4) == 1.0
    assert suco.recall([3, 7, 5, 6], truth, 4) == 0.5
    assert suco.recall([8, 5, 6, 4], truth, 4) == 0.0
    assert suco.recall([1, 9, 7, 3], truth, 4) == 1.0
    assert suco.recall([3, 7], truth, 4) == 0.5
    with pytest.raises(suco.ContractError):
        suco.recall([3], truth, 5)


def test_mre_known_answers(suco):  # test_eval.cpp:67-82
    truth = [1.0, 2.0]
    assert suco.mre([1.1, 2.2], truth, 2) == pytest.approx(0.1)
    assert suco.mre([1.0, 2.0], truth, 2) == pytest.approx(0.0)
    assert suco.mre([2.0, 2.0], truth, 2) == pytest.approx(0.5)
    assert suco.mre([1.0, 2.2], [0.0, 2.0], 2) == pytest.approx(0.1)
    assert suco.mre([0.0, 0.0], [0.0, 0.0], 2) == 0.0
    assert math.isinf(suco.mre([1.0, 1.0], [0.0, 0.0], 2))


@pytest.mark.gpu
@pytest.mark.parametrize("quant,k", [(True, 10), (False, 10), (True, 40), (False, 1), (True, 1)])
def test_exact_knn_matches_reference(gpu, oracle, ref, quant, k):
    full = oracle.clustered(3000 + 20, 20, 15, 77 + k, 0, 200, 12, quant)
    base, qs = oracle.hold_out(full, 20, 78)
    idx = gpu.build_index(base, gpu.IndexParams(4, 8, 2, 42))
    ids, dd = idx.exact_knn_batch(qs, k)
    for i, q in enumerate(qs):
        wi, wd = ref.exact_knn(base, q, k)
        assert np.array_equal(ids[i], wi), (quant, k, i)
        assert np.array_equal(dd[i], wd), (quant, k, i)


@pytest.mark.gpu
def test_exact_knn_k_equals_n_and_errors(gpu, ref):  # test_eval.cpp:41-51
    rng = np.random.default_rng(3)
    base = rng.integers(0, 5, size=(40, 6)).astype(np.float32)  # many distance ties
    q = rng.integers(0, 5, size=(2, 6)).astype(np.float32)
    idx = gpu.build_index(base, gpu.IndexParams(2, 3, 2, 42))
    ids, dd = idx.exact_knn_batch(q, 40)
    for i in range(2):
        wi, wd = ref.exact_knn(base, q[i], 40)
        assert np.array_equal(ids[i], wi) and np.array_equal(dd[i], wd)
        assert sorted(ids[i].tolist()) == list(range(40))
    with pytest.raises(gpu.ContractError):
        idx.exact_knn_batch(q, 41)
    with pytest.raises(gpu.ContractError):
        idx.exact_knn_batch(q, 0)
    with pytest.raises(gpu.ContractError):
        idx.exact_knn_batch(q[:, :5], 3)


@pytest.mark.gpu
def test_recall_of_exhaustive_query_is_one(gpu, oracle):
    """alpha = beta = 1 makes knn_query exact (test_query.cpp:216-238): recall 1, mre 0."""
    full = oracle.clustered(2000 + 10, 16, 10, 5, 0, 100, 8, False)
    base, qs = oracle.hold_out(full, 10, 6)
    idx = gpu.build_index(base, gpu.IndexParams(4, 8, 2, 42))
    ids, dd = idx.knn_query_batch(qs, gpu.CollisionParams(1.0, 1.0, 10))
    ti, td = idx.exact_knn_batch(qs, 10)
    for i in range(len(qs)):
        assert gpu.recall(ids[i], ti[i], 10) == 1.0
        assert gpu.mre(dd[i], td[i], 10) == 0.0
