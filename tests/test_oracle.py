"""Pins the CPU oracle (oracle/suco_oracle.c) before anything is checked against it.

Sources of truth, in order:
  1. the reference's own known-answer tests (cited file:line),
  2. golden fixtures produced by the reference itself (tests/golden/make_golden.py),
  3. the reference library compiled from its sources (oracle/_ref), when present.
"""
import numpy as np
import pytest

from conftest import golden


# ------------------------------------------------------------------ KATs
def test_splitmix64_kat(oracle):  # test_rng_parallel.cpp:15-19
    assert oracle.splitmix64(0) == 0xE220A8397B1DCDAF
    assert oracle.splitmix64(1) == 0x910A2DEC89025CC1
    assert oracle.splitmix64(0xDEADBEEF) == 0x4ADFB90F68C9EB9B


def test_derive_seed_separates_streams(oracle):  # test_rng_parallel.cpp:21-29
    seen = {oracle.derive_seed(42, s) for s in range(64)}
    assert len(seen) == 64
    assert oracle.derive_seed(42, 3) == oracle.derive_seed(42, 3)
    assert oracle.derive_seed(42, 3) != oracle.derive_seed(43, 3)


def test_fnv1a_kat(oracle):  # test_core.cpp:75-79
    assert oracle.fnv1a(b"") == 0xCBF29CE484222325
    assert oracle.fnv1a(b"a") == 0xAF63DC4C8601EC8C


COLLISION_KATS = [  # test_sc_linear.cpp:15-29
    (0.05, 10000000, 500000), (0.05, 10, 1), (0.001, 100, 1), (0.0001, 100, 1), (0.75, 10, 7), (1.0, 42, 42),
    (0.7, 10, 7), (0.3, 10, 3), (0.07, 100, 7),
]
CANDIDATE_KATS = [  # test_sc_linear.cpp:31-38
    (0.005, 10000, 50, 50), (0.005, 100000, 50, 500), (0.0051, 10000, 10, 51), (1.0, 777, 10, 777),
    (0.001, 10000, 50, 50), (0.3, 10, 1, 3),
]


@pytest.mark.parametrize("alpha,n,want", COLLISION_KATS)
def test_collision_count_kat(oracle, alpha, n, want):
    assert oracle.collision_count(alpha, n) == want


@pytest.mark.parametrize("beta,n,k,want", CANDIDATE_KATS)
def test_candidate_count_kat(oracle, beta, n, k, want):
    assert oracle.candidate_count(beta, n, k) == want


def test_params_validation(oracle):  # test_sc_linear.cpp:40-59
    from oracle.oracle import OracleError
    oracle.validate_params(0.05, 0.005, 50, 1000)
    for bad in (0.0, -0.5, 1.5):
        with pytest.raises(OracleError) as e:
            oracle.validate_params(bad, 0.005, 50, 1000)
        assert e.value.code == 2
        with pytest.raises(OracleError) as e:
            oracle.validate_params(0.05, bad, 50, 1000)
        assert e.value.code == 2
    for k in (0, 1001):
        with pytest.raises(OracleError):
            oracle.validate_params(0.05, 0.005, k, 1000)
    oracle.validate_params(0.05, 0.005, 1000, 1000)


def test_imi_fixture(oracle):  # test_index.cpp:44-58
    off, ids = oracle.build_imi([0, 1, 0, 1], [0, 1, 0, 0], 2)
    assert off.tolist() == [0, 2, 2, 3, 4]
    assert ids.tolist() == [0, 2, 3, 1]


def test_build_imi_validates(oracle):  # test_index.cpp:60-66
    from oracle.oracle import OracleError
    with pytest.raises(OracleError) as e:
        oracle.build_imi([0, 1], [0, 2], 2)
    assert e.value.code == 5


def one_point_per_cell(oracle):
    return oracle.build_imi([0, 0, 1, 1], [0, 1, 0, 1], 2)[0]


def make_cd(d):
    d = np.asarray(d, np.float64)
    order = np.array(sorted(range(len(d)), key=lambda i: (d[i], i)), np.uint32)
    return d, order


@pytest.mark.parametrize("kind", [0, 2])
def test_traversal_hand_fixture(oracle, kind):  # test_query.cpp:71-88
    d1, o1 = make_cd([0.2, 0.4])
    d2, o2 = make_cd([0.5, 0.8])
    c1, c2, cum, sums = oracle.traverse(kind, 0.75, 4, d1, o1, d2, o2, 2, one_point_per_cell(oracle))
    assert list(zip(c1.tolist(), c2.tolist(), cum.tolist())) == [(0, 0, 1), (1, 0, 2), (0, 1, 3)]
    assert sums.tolist() == [0.2 + 0.5, 0.4 + 0.5, 0.2 + 0.8]


def test_traversal_rank_mapping(oracle):  # test_query.cpp:90-103
    d1, o1 = make_cd([0.4, 0.2])
    d2, o2 = make_cd([0.5, 0.8])
    c1, c2, cum, sums = oracle.traverse(0, 1.0, 4, d1, o1, d2, o2, 2, one_point_per_cell(oracle))
    assert (c1[0], c2[0]) == (1, 0) and cum[-1] == 4 and len(c1) == 4


def test_traversal_matches_reference_golden(oracle):
    """DA and the exhaustive sort-all-cells oracle equal the reference's DA on 56 random instances."""
    g = golden("traversal.npz")
    for i in range(int(g["count"][0])):
        k, n, alpha = g[f"t{i}_meta"]
        args = (alpha, int(n), g[f"t{i}_d1"], g[f"t{i}_o1"], g[f"t{i}_d2"], g[f"t{i}_o2"], int(k), g[f"t{i}_off"])
        for kind in (0, 2):
            c1, c2, cum, sums = oracle.traverse(kind, *args)
            assert np.array_equal(c1, g[f"t{i}_c1"]) and np.array_equal(c2, g[f"t{i}_c2"])
            assert np.array_equal(cum, g[f"t{i}_cum"]) and np.array_equal(sums, g[f"t{i}_sums"])


def test_centroid_distances_golden(oracle):
    g = golden("centroid_distances.npz")
    d, o = oracle.centroid_distances(g["q"], g["cent"], 50)
    assert np.array_equal(d, g["dists"]) and np.array_equal(o, g["order"])
    # test_query.cpp:53-69: true Euclidean, ties by id
    d, o = oracle.centroid_distances([2.0], [0.0, 3.0], 2)
    assert d.tolist() == [2.0, 1.0] and o.tolist() == [1, 0]
    assert oracle.centroid_distances([2.0], [1.0, 3.0], 2)[1].tolist() == [0, 1]


def test_rerank_golden(oracle):
    g = golden("rerank.npz")
    for j in range(3):
        ids, d = oracle.rerank(g["data"], g["queries"][j], g["cands"], 15)
        assert np.array_equal(ids, g[f"ids{j}"]) and np.array_equal(d, g[f"dists{j}"])


def test_kmeans_golden(oracle):
    g = golden("kmeans.npz")
    km = oracle.kmeans(g["pts"], 20, 8, 5)
    assert np.array_equal(km["centroids"], g["centroids"])
    assert np.array_equal(km["assignments"], g["assignments"])
    km2 = oracle.kmeans(g["dup"], 8, 5, 13)  # test_kmeans.cpp:93-110: forces empty-cluster repair
    assert np.array_equal(km2["centroids"], g["dup_centroids"])
    assert np.array_equal(km2["assignments"], g["dup_assignments"])
    assert np.array_equal(km2["repaired"], g["dup_repaired"]) and km2["repaired"].size > 0


def test_build_and_query_golden(oracle):
    g = golden("e2e_small.npz")
    idx = oracle.build_index(g["base"], 4, 12, 5, 42, 0)
    assert idx.serialize() == g["index"].tobytes()
    for tag in ("p0", "p1", "p2"):
        a, b, k = g[f"{tag}_params"]
        ids, d, _ = idx.knn_query_batch(g["base"], g["queries"], a, b, int(k), threads=2)
        assert np.array_equal(ids, g[f"{tag}_ids"]) and np.array_equal(d, g[f"{tag}_dists"])
    scores, cands, cps, cum = idx.query_intermediates(g["base"], g["queries"][0], 0.05, 0.05, 10)
    assert np.array_equal(scores, g["scores_q0"]) and np.array_equal(cands, g["cands_q0"])
    assert np.array_equal(cps, g["cells_q0"]) and np.array_equal(cum, g["cum_q0"])


def test_shuffled_layout_golden(oracle):
    g = golden("e2e_shuffled.npz")
    idx = oracle.build_index(g["base"], 3, 7, 4, 9, 1)
    assert idx.serialize() == g["index"].tobytes()
    a, b, k = g["params"]
    ids, d, _ = idx.knn_query_batch(g["base"], g["queries"], a, b, int(k))
    assert np.array_equal(ids, g["ids"]) and np.array_equal(d, g["dists"])


def test_deserialize_roundtrip_and_corruption(oracle):
    from oracle.oracle import OracleError
    blob = golden("e2e_small.npz")["index"].tobytes()
    assert oracle.load_index(blob).serialize() == blob
    for cut in (0, 3, 4, 10, 47, 60, len(blob) // 2, len(blob) - 1):  # test_index.cpp:156-208
        with pytest.raises(OracleError) as e:
            oracle.load_index(blob[:cut])
        assert e.value.code == 3
    with pytest.raises(OracleError):
        oracle.load_index(b"SUCX" + blob[4:])
    with pytest.raises(OracleError):
        oracle.load_index(blob + b"\0")


# ------------------------------------------------- against the live reference
def test_generators_match_reference(oracle, ref):
    assert np.array_equal(oracle.clustered(500, 24, 7, 3, 0, 100, 5, False), ref.clustered(500, 24, 7, 3, 0, 100, 5, False))
    assert np.array_equal(oracle.uniform(300, 16, 41), ref.uniform(300, 16, 41))
    a = oracle.clustered(300, 16, 9, 5, 20, 140, 18, True)
    assert np.array_equal(a, ref.clustered(300, 16, 9, 5, 20, 140, 18, True))
    ba, qa = oracle.hold_out(a, 30, 8)
    bb, qb = ref.hold_out(a, 30, 8)
    assert np.array_equal(ba, bb) and np.array_equal(qa, qb)
    for mode in (0, 1):
        lo, lr = oracle.sample_subspaces(22, 3, mode, 9), ref.sample_subspaces(22, 3, mode, 9)
        assert np.array_equal(lo.dims, lr.dims) and np.array_equal(lo.sizes, lr.sizes)


@pytest.mark.parametrize("seed", [101, 102, 103])
def test_random_builds_match_reference(oracle, ref, seed):
    data = oracle.clustered(1500, 16, 8, seed, 0.0, 100.0, 10.0, False)
    qs = oracle.uniform(25, 16, seed + 1, 0.0, 100.0)
    io = oracle.build_index(data, 4, 20, 5, seed, 0)
    ir = ref.build_index(data, 4, 20, 5, seed, 0)
    assert io.serialize() == ir.serialize()
    for a, b, k in ((0.05, 0.01, 10), (1.0, 1.0, 10), (0.3, 0.002, 3)):
        i1, d1, _ = io.knn_query_batch(data, qs, a, b, k)
        i2, d2, _ = ir.knn_query_batch(data, qs, a, b, k, threads=2)
        assert np.array_equal(i1, i2) and np.array_equal(d1, d2)


# ------------------------------- config 5's sampled build (no reference API; pinned by composition)
def _sampled_case(oracle, seed, n=2400, d=16, ns=4, k_half=12, n_train=500, quantize=False, mode=0):
    data = oracle.clustered(n, d, 9, seed, 0.0, 100.0, 10.0, quantize)
    train = np.sort(np.random.default_rng(seed).choice(n, n_train, replace=False)).astype(np.uint32)
    return data, train, dict(ns=ns, k_half=k_half, iters=4, seed=seed, mode=mode)


def test_sampled_build_with_every_row_is_build_index(oracle):
    data, _, p = _sampled_case(oracle, 31)
    full = np.arange(data.shape[0], dtype=np.uint32)
    a = oracle.build_index_sampled(data, full, p["ns"], p["k_half"], p["iters"], p["seed"], p["mode"]).serialize()
    assert a == oracle.build_index(data, p["ns"], p["k_half"], p["iters"], p["seed"], p["mode"]).serialize()


@pytest.mark.parametrize("seed,quantize,mode", [(41, False, 0), (42, True, 0), (43, False, 1)])
def test_sampled_build_pinned_to_reference(oracle, ref, seed, quantize, mode):
    """Centroids = the reference's build_index over the training rows (same jobs, same seeds);
    each training row's cell = its cell in that reference index; every other row's half-subspace
    cell = the first entry of the reference's own centroid_distances order (query.cpp:42-64)."""
    from suco_bytes import cell_of, parse

    data, train, p = _sampled_case(oracle, seed, quantize=quantize, mode=mode)
    mine = parse(oracle.build_index_sampled(data, train, p["ns"], p["k_half"], p["iters"], p["seed"], p["mode"])
                 .serialize())
    theirs = parse(ref.build_index(data[train], p["ns"], p["k_half"], p["iters"], p["seed"], p["mode"]).serialize())
    n, kh = data.shape[0], p["k_half"]
    assert mine["n"] == n and theirs["n"] == train.size
    others = np.setdiff1d(np.arange(n), train)[::23]
    for s in range(p["ns"]):
        a, b = mine["subspaces"][s], theirs["subspaces"][s]
        assert np.array_equal(a["cent1"], b["cent1"]) and np.array_equal(a["cent2"], b["cent2"])
        ca, cb = cell_of(a, n), cell_of(b, train.size)
        assert np.array_equal(ca[train], cb)
        dims = mine["dims"][s]
        h1 = len(dims) // 2
        for i in others:
            row = data[i, dims]
            _, o1 = ref.centroid_distances(row[:h1], a["cent1"], kh)
            _, o2 = ref.centroid_distances(row[h1:], a["cent2"], kh)
            assert ca[i] == int(o1[0]) * kh + int(o2[0])


def test_sampled_build_validation(oracle):
    from oracle.oracle import OracleError

    data, train, p = _sampled_case(oracle, 51)
    args = (p["ns"], p["k_half"], p["iters"], p["seed"], p["mode"])
    with pytest.raises(OracleError) as e:  # fewer training rows than k_half -> ConfigError
        oracle.build_index_sampled(data, train[: p["k_half"] - 1], *args)
    assert e.value.code == 2
    oracle.build_index_sampled(data, train[: p["k_half"]], *args)  # exactly k_half trains
    for bad in (train[::-1].copy(), np.array([0, 0] + list(range(2, 40)), np.uint32),
                np.array(list(range(30)) + [data.shape[0]], np.uint32)):
        with pytest.raises(OracleError) as e:  # not strictly ascending / out of range -> ContractError
            oracle.build_index_sampled(data, bad, *args)
        assert e.value.code == 5
