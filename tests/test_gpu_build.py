"""GPU index build parity: k-means, IMI and whole indexes byte-identical to the reference."""
import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def test_kmeans_golden(gpu):
    g = golden("kmeans.npz")
    km = gpu.kmeans(g["pts"], 20, 8, 5)  # test_kmeans.cpp:70-83 shape
    assert np.array_equal(km["centroids"], g["centroids"])
    assert np.array_equal(km["assignments"], g["assignments"])
    km2 = gpu.kmeans(g["dup"], 8, 5, 13)  # test_kmeans.cpp:93-110: empty clusters repaired
    assert np.array_equal(km2["centroids"], g["dup_centroids"])
    assert np.array_equal(km2["assignments"], g["dup_assignments"])
    assert np.array_equal(km2["repaired"], g["dup_repaired"]) and km2["repaired"].size > 0
    assert km2["assignments"][0] != km2["assignments"][1]


@pytest.mark.parametrize("n,dim,k,iters,kind", [(5000, 8, 50, 4, "int"), (3000, 6, 64, 3, "float"),
                                                (4000, 30, 50, 2, "float"), (2000, 3, 7, 5, "unit"),
                                                (600, 4, 3, 10, "float"), (12, 2, 12, 3, "float"),
                                                (20000, 8, 100, 2, "int"), (800, 40, 10, 3, "int"),
                                                (60000, 4, 20, 2, "dyadic"), (50000, 6, 16, 2, "float"),
                                                (30000, 2, 9, 2, "huge"), (300000, 4, 16, 2, "dyadic"),
                                                (400000, 6, 24, 2, "float"), (300000, 2, 9, 2, "huge"),
                                                (250000, 5, 12, 2, "unit"), (200000, 8, 20, 1, "int")])
def test_kmeans_vs_oracle(gpu, oracle, n, dim, k, iters, kind):
    """Exact k-means against the restated reference. "dyadic" (quarter-integers plus halves: few
    mantissa bits, so the running k-means++ sum meets exact rounding ties) and "huge" (magnitudes
    spanning 1e-30..1e30: binade crossings and serial adds everywhere) stress the parallel exact
    fold of the k-means++ sums; the larger float corpora cross many binades. Corpora past 32,768
    points span several fold chunks (build.cu kpp_chunk_fold_kernel: per-chunk integer sums under
    the predicted binade, look-back of the exact running sum, tile scans for the crossing chunks)."""
    rng = np.random.default_rng(n + dim + k)
    if kind == "int":
        pts = np.clip(np.rint(rng.normal(100, 30, (n, dim))), 0, 255).astype(np.float32)
    elif kind == "unit":
        pts = rng.random((n, dim)).astype(np.float32)
    elif kind == "dyadic":
        pts = (np.rint(rng.normal(0, 40, (n, dim))) / 4 + 0.5).astype(np.float32)
    elif kind == "huge":
        pts = (rng.normal(0, 1, (n, dim)) * 10.0 ** rng.integers(-15, 15, (n, 1))).astype(np.float32)
    else:
        pts = (rng.normal(0, 1, (n, dim)) * 10).astype(np.float32)
    for seed in (1, 99):
        a = gpu.kmeans(pts, k, iters, seed)
        b = oracle.kmeans(pts, k, iters, seed)
        assert np.array_equal(a["centroids"], b["centroids"]), (kind, seed)
        assert np.array_equal(a["assignments"], b["assignments"]), (kind, seed)
        assert np.array_equal(a["repaired"], b["repaired"]), (kind, seed)


def test_kmeans_k_equals_n(gpu):  # test_kmeans.cpp:112-119
    pts = np.random.default_rng(3).random((12, 2)).astype(np.float32)
    km = gpu.kmeans(pts, 12, 3, 9)
    assert len(set(km["assignments"].tolist())) == 12


def test_kmeans_validation(gpu):  # test_kmeans.cpp:121-126
    pts = np.zeros((10, 2), np.float32)
    for k, it in ((0, 5), (3, 0), (11, 5)):
        with pytest.raises(gpu.ConfigError):
            gpu.kmeans(pts, k, it, 1)


def test_build_imi(gpu, oracle):  # test_index.cpp:44-74
    off, ids = gpu.build_imi([0, 1, 0, 1], [0, 1, 0, 0], 2)
    assert off.tolist() == [0, 2, 2, 3, 4] and ids.tolist() == [0, 2, 3, 1]
    rng = np.random.default_rng(15)
    for k_half in (1, 2, 7, 32, 120):
        a, b = rng.integers(0, k_half, 5000), rng.integers(0, k_half, 5000)
        o1, i1 = gpu.build_imi(a, b, k_half)
        o2, i2 = oracle.build_imi(a, b, k_half)
        assert np.array_equal(o1, o2) and np.array_equal(i1, i2)
    with pytest.raises(gpu.ContractError):
        gpu.build_imi([0, 1], [0, 2], 2)
    with pytest.raises(gpu.ContractError):
        gpu.build_imi([0, 1], [0], 2)


def test_build_index_golden(gpu):
    g = golden("e2e_small.npz")
    idx = gpu.build_index(g["base"], gpu.IndexParams(4, 12, 5, 42))
    assert idx.serialize() == g["index"].tobytes()
    ids, d = idx.knn_query_batch(g["queries"], gpu.CollisionParams(0.05, 0.05, 10))
    assert np.array_equal(ids, g["p0_ids"]) and np.array_equal(d, g["p0_dists"])


def test_build_index_shuffled_golden(gpu):
    g = golden("e2e_shuffled.npz")
    idx = gpu.build_index(g["base"], gpu.IndexParams(3, 7, 4, 9, gpu.SubspaceMode.Shuffled))
    assert idx.serialize() == g["index"].tobytes()


@pytest.mark.parametrize("case", [
    (3000, 32, 20, 0, 100, 8, False, 4, 16, 4, 0),
    (5000, 16, 30, 20, 140, 18, True, 2, 40, 3, 1),
    (2000, 60, 10, 0, 1, 0.05, False, 3, 10, 2, 0),
    (1500, 16, 8, 0, 100, 10, False, 8, 20, 5, 0),
])
def test_build_index_vs_oracle(gpu, oracle, case):
    n, d, cl, lo, hi, sig, q, ns, kh, it, mode = case
    data = oracle.clustered(n, d, cl, n + d, lo, hi, sig, q)
    ours = gpu.build_index(data, gpu.IndexParams(ns, kh, it, 7, gpu.SubspaceMode(mode)))
    theirs = oracle.build_index(data, ns, kh, it, 7, mode)
    assert ours.serialize() == theirs.serialize()


def test_build_index_vs_reference(gpu, ref):
    """The reference's own build_index on a descriptor corpus (acceptance.cpp:70-74 shape)."""
    full = ref.clustered(10100, 128, 64, 7, 20.0, 140.0, 18.0, True)
    base, queries = ref.hold_out(full, 100, 8)
    ours = gpu.build_index(base, gpu.IndexParams())
    theirs = ref.build_index(base, 8, 50, 10, 42, 0)
    assert ours.serialize() == theirs.serialize()
    ids, d = ours.knn_query_batch(queries, gpu.CollisionParams(0.05, 0.05, 50))
    ri, rd, _ = theirs.knn_query_batch(base, queries, 0.05, 0.05, 50)
    assert np.array_equal(ids, ri) and np.array_equal(d, rd)


def test_build_index_errors(gpu):  # index.cpp:100-111, subspace.cpp:12-21, core.cpp:8-21
    data = np.random.default_rng(0).random((100, 8)).astype(np.float32)
    for p in (gpu.IndexParams(2, 0, 3), gpu.IndexParams(2, 5, 0), gpu.IndexParams(2, 101, 3),
              gpu.IndexParams(1, 5, 3), gpu.IndexParams(5, 5, 3)):
        with pytest.raises(gpu.ConfigError):
            gpu.build_index(data, p)
    bad = data.copy()
    bad[3, 1] = np.inf
    with pytest.raises(gpu.ContractError):
        gpu.build_index(bad, gpu.IndexParams(2, 5, 3))


# ---------------------------------------- config 5's sampled build (suco_gpu_build_index_sampled)
@pytest.mark.parametrize("case", [
    # n, d, clusters, lo, hi, sigma, quantize, ns, k_half, iters, mode, n_train, chunk
    (6000, 32, 20, 0, 100, 8, False, 4, 16, 4, 0, 700, None),
    (8000, 16, 30, 20, 140, 18, True, 2, 40, 3, 1, 1200, 999),     # several assignment chunks, ragged last
    (3000, 60, 10, 0, 1, 0.05, False, 3, 10, 2, 0, 10, 3000),      # n_train == k_half; h = 10
    (2500, 16, 8, 0, 100, 10, False, 8, 20, 5, 0, 2500, None),     # every row trains
])
def test_sampled_build_vs_oracle(gpu, oracle, monkeypatch, case):
    n, d, cl, lo, hi, sig, q, ns, kh, it, mode, nt, chunk = case
    if chunk:
        monkeypatch.setenv("SUCO_BUILD_CHUNK", str(chunk))
    data = oracle.clustered(n, d, cl, n + d, lo, hi, sig, q)
    train = np.sort(np.random.default_rng(n).choice(n, nt, replace=False)).astype(np.uint32)
    ours = gpu.build_index_sampled(data, train, gpu.IndexParams(ns, kh, it, 7, gpu.SubspaceMode(mode)))
    theirs = oracle.build_index_sampled(data, train, ns, kh, it, 7, mode)
    assert ours.serialize() == theirs.serialize()


def test_sampled_build_from_device_rows(gpu, oracle):
    torch = pytest.importorskip("torch")
    data = oracle.clustered(5000, 24, 12, 5, 0, 100, 8, False)
    train = np.arange(0, 5000, 7, dtype=np.uint32)
    p = gpu.IndexParams(3, 16, 3, 11)
    host = gpu.build_index_sampled(data, train, p).serialize()
    dev = torch.from_numpy(data).cuda()
    assert gpu.build_index_sampled(dev, train, p).serialize() == host
    assert gpu.build_index(dev, p).serialize() == gpu.build_index(data, p).serialize()


def test_sampled_build_errors(gpu):
    data = np.random.default_rng(0).random((300, 8)).astype(np.float32)
    p = gpu.IndexParams(2, 5, 3)
    with pytest.raises(gpu.ConfigError):  # fewer training rows than k_half
        gpu.build_index_sampled(data, np.arange(4), p)
    for bad in (np.arange(10)[::-1], np.array([1, 1, 2, 3, 4, 5]), np.array([0, 1, 2, 3, 4, 300])):
        with pytest.raises(gpu.ContractError):
            gpu.build_index_sampled(data, bad, p)
    nan = data.copy()
    nan[5, 2] = np.nan
    with pytest.raises(gpu.ContractError):  # dataset invariants first (core.cpp:15-19)
        gpu.build_index_sampled(nan, np.arange(50), p)


def test_sampled_cfg5_shape_query_vs_reference(gpu, ref):
    """Config 5's shape scaled down (u8 descriptors, N_s = 8, 100 x 100 centroids on a 1 % sample,
    alpha = 0.02, beta = 0.002): K = 10,000 cells per subspace takes the half-width dense select (u16 masks, two points per lane).
    The reference's own load_index + knn_query on the GPU-built bytes give the same answers."""
    import bench_data

    cfg = bench_data.CONFIGS["cfg5"]
    base, queries = bench_data.generate(cfg, n=300_000, queries=48)
    train = bench_data.train_ids(cfg, base.shape[0])
    idx = gpu.build_index_sampled(base, train, gpu.IndexParams(8, 100, 10, 42))
    blob = idx.serialize()
    cp = gpu.CollisionParams(cfg.alpha, cfg.beta, cfg.k)
    ids, dists = idx.knn_query_batch(queries, cp)
    ri, rd, _ = ref.load_index(blob).knn_query_batch(base, queries, cfg.alpha, cfg.beta, cfg.k)
    assert np.array_equal(ids, ri) and np.array_equal(dists, rd)
