"""GPU parity of the query path against the oracle and the reference's golden outputs.

Bar (BASELINE.json north_star): identical retrieved cells, SC-scores, candidate
sets and top-k ids; distances bit-identical here (stricter than the stated
1e-5 relative tolerance, which TOL below records for the record).
"""
import os

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu
TOL = 1e-5  # north_star tolerance on distances; every check below is exact equality


def make_cd(d):
    d = np.asarray(d, np.float64)
    return d, np.array(sorted(range(len(d)), key=lambda i: (d[i], i)), np.uint32)


def cells_equal(got, c1, c2, cum, sums):
    assert len(got) == len(c1)
    assert [g.c1 for g in got] == c1.tolist()
    assert [g.c2 for g in got] == c2.tolist()
    assert [g.cumulative for g in got] == cum.tolist()
    assert np.array_equal(np.array([g.sum_dist for g in got], np.float64), sums)


# ------------------------------------------------------------ stage: centroids
def test_centroid_distances(gpu):
    g = golden("centroid_distances.npz")
    d, o = gpu.centroid_distances(g["q"], g["cent"], 50)
    assert np.array_equal(d, g["dists"]) and np.array_equal(o, g["order"])
    d, o = gpu.centroid_distances([2.0], [0.0, 3.0], 2)  # test_query.cpp:53-69
    assert d.tolist() == [2.0, 1.0] and o.tolist() == [1, 0]
    assert gpu.centroid_distances([2.0], [1.0, 3.0], 2)[1].tolist() == [0, 1]
    with pytest.raises(gpu.ContractError):
        gpu.centroid_distances([2.0], [0.0, 3.0], 3)


@pytest.mark.parametrize("k,h", [(50, 8), (64, 6), (100, 30), (7, 3), (300, 5)])
def test_centroid_distances_vs_oracle(gpu, oracle, k, h):
    rng = np.random.default_rng(k * 31 + h)
    cent = rng.integers(0, 6, size=(k, h)).astype(np.float32)  # coarse grid: many exact ties
    q = rng.integers(0, 6, size=h).astype(np.float32)
    d1, o1 = gpu.centroid_distances(q, cent, k)
    d2, o2 = oracle.centroid_distances(q, cent, k)
    assert np.array_equal(d1, d2) and np.array_equal(o1, o2)


# ------------------------------------------------------------ stage: traversal
def test_traversal_hand_fixture(gpu, oracle):  # test_query.cpp:71-88
    off = oracle.build_imi([0, 0, 1, 1], [0, 1, 0, 1], 2)[0]
    r = gpu.dynamic_activation(0.75, 4, make_cd([0.2, 0.4]), make_cd([0.5, 0.8]), off)
    assert [(c.c1, c.c2, c.cumulative) for c in r] == [(0, 0, 1), (1, 0, 2), (0, 1, 3)]
    assert [c.sum_dist for c in r] == [0.2 + 0.5, 0.4 + 0.5, 0.2 + 0.8]
    r = gpu.dynamic_activation(1.0, 4, make_cd([0.4, 0.2]), make_cd([0.5, 0.8]), off)  # :90-103
    assert (r[0].c1, r[0].c2) == (1, 0) and r[-1].cumulative == 4 and len(r) == 4


def test_traversal_golden(gpu):
    """56 random instances incl. quantised ties: identical to the reference's DA."""
    g = golden("traversal.npz")
    for i in range(int(g["count"][0])):
        k, n, alpha = g[f"t{i}_meta"]
        got = gpu.dynamic_activation(alpha, int(n), (g[f"t{i}_d1"], g[f"t{i}_o1"]), (g[f"t{i}_d2"], g[f"t{i}_o2"]),
                                     g[f"t{i}_off"])
        cells_equal(got, g[f"t{i}_c1"], g[f"t{i}_c2"], g[f"t{i}_cum"], g[f"t{i}_sums"])


@pytest.mark.parametrize("k_half,n,alpha,quant", [(33, 3000, 0.2, True), (100, 20000, 0.05, False),
                                                  (200, 5000, 0.3, True), (300, 9000, 0.02, False),
                                                  (1024, 200000, 0.005, False)])
def test_traversal_vs_oracle(gpu, oracle, k_half, n, alpha, quant):
    rng = np.random.default_rng(k_half + n)

    def cd():
        d = (rng.integers(0, 10, k_half) * 0.1) if quant else rng.random(k_half)
        return make_cd(d)

    off = oracle.build_imi(rng.integers(0, k_half, n), rng.integers(0, k_half, n), k_half)[0]
    cd1, cd2 = cd(), cd()
    got = gpu.dynamic_activation(alpha, n, cd1, cd2, off)
    want = oracle.traverse(0, alpha, n, cd1[0], cd1[1], cd2[0], cd2[1], k_half, off)
    cells_equal(got, *want)
    assert got[-1].cumulative >= gpu.collision_count(alpha, n)


def test_traversal_validation(gpu, oracle):  # test_query.cpp:175-186
    rng = np.random.default_rng(5)
    off = oracle.build_imi(rng.integers(0, 4, 20), rng.integers(0, 4, 20), 4)[0]
    cd1, cd2 = make_cd(rng.random(4)), make_cd(rng.random(4))
    for bad_alpha in (0.0, 1.5):
        with pytest.raises(gpu.ContractError):
            gpu.dynamic_activation(bad_alpha, 20, cd1, cd2, off)
    with pytest.raises(gpu.ContractError):
        gpu.dynamic_activation(0.5, 21, cd1, cd2, off)
    with pytest.raises(gpu.ContractError):
        gpu.dynamic_activation(0.5, 20, make_cd(rng.random(3)), cd2, off)


# ------------------------------------------------------------ stage: rerank
def test_rerank_golden(gpu):
    g = golden("rerank.npz")
    for j in range(3):
        r = gpu.rerank(g["data"], g["queries"][j], g["cands"], 15)
        assert [x.id for x in r] == g[f"ids{j}"].tolist()
        assert np.array_equal(np.array([x.distance for x in r]), g[f"dists{j}"])


@pytest.mark.parametrize("n,d,m,k", [(500, 128, 300, 10), (700, 22, 500, 7), (300, 3, 200, 5), (400, 960, 130, 32),
                                     (900, 96, 800, 40), (64, 16, 64, 64), (2000, 8, 1500, 1)])
def test_rerank_vs_oracle(gpu, oracle, n, d, m, k):
    rng = np.random.default_rng(n + d)
    data = rng.integers(0, 4, size=(n, d)).astype(np.float32)  # coarse values: distance ties
    q = rng.integers(0, 4, size=d).astype(np.float32)
    cands = rng.permutation(n)[:m].astype(np.uint32)
    r = gpu.rerank(data, q, cands, k)
    ids, dd = oracle.rerank(data, q, cands, k)
    assert [x.id for x in r] == ids.tolist()
    assert np.array_equal(np.array([x.distance for x in r]), dd)


def test_rerank_validation(gpu):  # test_query.cpp:207-213
    g = golden("rerank.npz")
    with pytest.raises(gpu.ContractError):
        gpu.rerank(g["data"], g["queries"][0], [1, 2, 3], 4)
    with pytest.raises(gpu.ContractError):
        gpu.rerank(g["data"], g["queries"][0], [1, 2, 3], 0)
    with pytest.raises(gpu.ContractError):
        gpu.rerank(g["data"], g["queries"][0], [1, 200], 1)
    with pytest.raises(gpu.ContractError):
        gpu.rerank(g["data"], np.zeros(6, np.float32), [1, 2, 3], 2)


# ------------------------------------------------------------ end to end
def test_knn_golden_small(gpu):
    g = golden("e2e_small.npz")
    idx = gpu.load_index(g["index"].tobytes(), g["base"])
    assert idx.serialize() == g["index"].tobytes()
    for tag in ("p0", "p1", "p2"):
        a, b, k = g[f"{tag}_params"]
        ids, d = idx.knn_query_batch(g["queries"], gpu.CollisionParams(a, b, int(k)))
        assert np.array_equal(ids, g[f"{tag}_ids"]), tag
        assert np.array_equal(d, g[f"{tag}_dists"]), tag
        assert np.allclose(d, g[f"{tag}_dists"], rtol=TOL, atol=0)


def test_intermediates_golden(gpu):
    g = golden("e2e_small.npz")
    idx = gpu.load_index(g["index"].tobytes(), g["base"])
    scores, cands, cps, cum = idx.query_intermediates(g["queries"][0], gpu.CollisionParams(0.05, 0.05, 10))
    assert np.array_equal(scores, g["scores_q0"])
    assert np.array_equal(cands, g["cands_q0"])
    assert np.array_equal(cps, g["cells_q0"]) and np.array_equal(cum, g["cum_q0"])
    assert int(scores.sum()) == int(cum.sum())  # each retrieved id scores once per subspace


def test_knn_golden_shuffled(gpu):
    g = golden("e2e_shuffled.npz")
    idx = gpu.load_index(g["index"].tobytes(), g["base"])
    a, b, k = g["params"]
    ids, d = idx.knn_query_batch(g["queries"], gpu.CollisionParams(a, b, int(k)))
    assert np.array_equal(ids, g["ids"]) and np.array_equal(d, g["dists"])


CASES = {
    # name: (n, d, clusters, lo, hi, sigma, quant, ns, k_half, iters, mode, [(alpha, beta, k)])
    "sift_like": (6000, 32, 30, 20, 140, 18, True, 4, 16, 4, 0, [(0.05, 0.005, 10), (0.02, 0.05, 50), (0.3, 0.001, 1)]),
    "float": (4000, 24, 20, 0, 1, 0.05, False, 3, 12, 3, 1, [(0.05, 0.01, 10), (0.5, 0.2, 33)]),
    "ns16": (3000, 64, 10, 0, 100, 8, False, 16, 6, 3, 0, [(0.05, 0.01, 10), (0.1, 0.004, 12)]),
    "ns40": (1200, 80, 10, 0, 100, 8, True, 40, 3, 2, 0, [(0.05, 0.05, 10)]),
    "tiny_touch": (2500, 16, 8, 0, 50, 3, False, 2, 8, 3, 0, [(0.0005, 0.4, 10), (0.001, 1.0, 25)]),
    # 64 x 64 cells: 128 KB of dense-select masks -> the 1024-thread, 1 CTA/SM variant
    "dense_1024": (20000, 32, 40, 0, 100, 8, False, 8, 64, 2, 0, [(0.05, 0.005, 10), (0.02, 0.05, 40)]),
    # 100 x 100 cells: the 128-leaf merge tree of the thread-per-task traversal
    "k100": (12000, 16, 20, 0, 100, 8, False, 2, 100, 2, 1, [(0.05, 0.01, 10), (0.2, 0.003, 5)]),
}


@pytest.mark.parametrize("trav", ["warp", "thread", "split", "nosplit", "ranked"])
@pytest.mark.parametrize("case", list(CASES))
def test_knn_vs_oracle(gpu, oracle, case, trav, monkeypatch):
    """Both traversal kernels (warp per task; thread per task with the merge tree, which large batches
    use) against the reference, cell order and cumulative sizes included."""
    monkeypatch.setenv("SUCO_TRAVERSE", trav)
    n, d, cl, lo, hi, sig, quant, ns, kh, it, mode, plist = CASES[case]
    full = oracle.clustered(n + 40, d, cl, 1000 + n, lo, hi, sig, quant)
    base, qs = oracle.hold_out(full, 40, 1001 + n)
    oidx = oracle.build_index(base, ns, kh, it, 42, mode)
    idx = gpu.load_index(oidx.serialize(), base)
    for a, b, k in plist:
        ids, dd = idx.knn_query_batch(qs, gpu.CollisionParams(a, b, k))
        oi, od, _ = oidx.knn_query_batch(base, qs, a, b, k)
        assert np.array_equal(ids, oi), (case, a, b, k)
        assert np.array_equal(dd, od), (case, a, b, k)
    for qi in (0, 7):
        a, b, k = plist[0]
        s1, c1, p1, u1 = idx.query_intermediates(qs[qi], gpu.CollisionParams(a, b, k))
        s2, c2, p2, u2 = oidx.query_intermediates(base, qs[qi], a, b, k)
        assert np.array_equal(s1, s2) and np.array_equal(c1, c2)
        assert np.array_equal(p1, p2) and np.array_equal(u1, u2)


def test_exhaustive_degeneracy(gpu, oracle, ref):
    """alpha = beta = 1 equals exact kNN (test_query.cpp:216-238, acceptance.cpp:87-136)."""
    data = oracle.clustered(300, 16, 4, 19, 0.0, 20.0, 2.0, False)
    qs = oracle.uniform(5, 16, 20, 0.0, 20.0)
    idx = gpu.load_index(oracle.build_index(data, 4, 5, 3, 42, 0).serialize(), data)
    ids, dd = idx.knn_query_batch(qs, gpu.CollisionParams(1.0, 1.0, 10))
    for qi in range(5):
        ei, ed = ref.exact_knn(data, qs[qi], 10)
        assert np.array_equal(ids[qi], ei) and np.array_equal(dd[qi], ed)


def test_self_query_returns_itself(gpu, oracle):  # test_query.cpp:262-282
    data = oracle.clustered(400, 16, 4, 31, 0.0, 40.0, 3.0, False)
    idx = gpu.load_index(oracle.build_index(data, 4, 8, 4, 42, 0).serialize(), data)
    ids, dd = idx.knn_query_batch(data[[0, 137, 399]], gpu.CollisionParams(0.1, 0.05, 5))
    for row, pid in enumerate((0, 137, 399)):
        assert dd[row, 0] == 0.0 and ids[row, 0] <= pid


@pytest.mark.parametrize("cluster", ["1", "2", "4", "16"])
def test_cluster_sizes_and_multi_round(gpu, oracle, cluster, monkeypatch):
    """Every cluster size, and the two-pass (rounds > 1) select, give identical results."""
    monkeypatch.setenv("SUCO_CLUSTER", cluster)
    n = 230000 if cluster == "1" else 60000  # CS = 1 and n > 200 KiB of counters: 2 rounds
    full = oracle.clustered(n + 16, 8, 64, 7, 0, 100, 6, True)
    base, qs = oracle.hold_out(full, 16, 8)
    oidx = oracle.build_index(base, 2, 16, 2, 42, 0)
    idx = gpu.load_index(oidx.serialize(), base)
    for a, b, k in ((0.05, 0.005, 10), (0.01, 0.02, 20)):
        ids, dd = idx.knn_query_batch(qs, gpu.CollisionParams(a, b, k))
        oi, od, _ = oidx.knn_query_batch(base, qs, a, b, k)
        assert np.array_equal(ids, oi) and np.array_equal(dd, od)
    s1, c1, _, _ = idx.query_intermediates(qs[3], gpu.CollisionParams(0.05, 0.005, 10))
    s2, c2, _, _ = oidx.query_intermediates(base, qs[3], 0.05, 0.005, 10)
    assert np.array_equal(s1, s2) and np.array_equal(c1, c2)


def test_device_batch_api(gpu):
    torch = pytest.importorskip("torch")
    g = golden("e2e_small.npz")
    idx = gpu.load_index(g["index"].tobytes(), g["base"])
    q = torch.from_numpy(g["queries"]).cuda()
    ids = torch.empty((q.shape[0], 10), dtype=torch.int32, device="cuda")
    dd = torch.empty((q.shape[0], 10), dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    idx.knn_query_batch_device(q.data_ptr(), q.shape[0], q.shape[1], gpu.CollisionParams(0.05, 0.05, 10),
                               ids.data_ptr(), dd.data_ptr(), s.cuda_stream)
    s.synchronize()
    assert np.array_equal(ids.cpu().numpy().view(np.uint32), g["p0_ids"])
    assert np.array_equal(dd.cpu().numpy(), g["p0_dists"])


def test_query_errors(gpu):  # test_query.cpp:314-332, query.cpp:202-208
    g = golden("e2e_small.npz")
    idx = gpu.load_index(g["index"].tobytes(), g["base"])
    with pytest.raises(gpu.ContractError):
        idx.knn_query_batch(np.zeros((1, 31), np.float32), gpu.CollisionParams())
    for bad in (gpu.CollisionParams(alpha=0.0), gpu.CollisionParams(beta=1.5), gpu.CollisionParams(k=0),
                gpu.CollisionParams(k=10**7)):
        with pytest.raises(gpu.ConfigError):
            idx.knn_query_batch(g["queries"][:1], bad)
    with pytest.raises(gpu.IncompatibilityError):
        gpu.knn_query(idx, g["base"][:-1], g["queries"][0], gpu.CollisionParams())


def test_load_errors(gpu):
    g = golden("e2e_small.npz")
    blob = g["index"].tobytes()
    with pytest.raises(gpu.IncompatibilityError):
        gpu.load_index(blob, g["base"][:-1])
    with pytest.raises(gpu.IncompatibilityError):
        gpu.load_index(blob, g["base"][:, :-1])
    for cut in (0, 4, 40, len(blob) // 3, len(blob) - 1):
        with pytest.raises(gpu.CorruptIndexError):
            gpu.load_index(blob[:cut], g["base"])
    bad = g["base"].copy()
    bad[5, 3] = np.nan
    with pytest.raises(gpu.ContractError, match="component 163 is not finite"):
        gpu.load_index(blob, bad)


@pytest.mark.gpu
@pytest.mark.parametrize("d,shift", [(40, 0.0), (128, 0.0), (17, 0.0), (40, -128.0)])
def test_u8_rows_rerank_mixed_queries(gpu, oracle, d, shift):
    """u8-valued rows take the byte re-rank (rerank_u8_kernel) for integer queries and the
    fp32/fp64 chains for the others, in the same batch; negative integers take no byte path."""
    full = oracle.clustered(5000 + 40, d, 25, 300 + d, 10, 240, 14, True)
    base, qs = oracle.hold_out(full, 40, 301 + d)
    base = (base + np.float32(shift)).astype(np.float32)
    qs = (qs + np.float32(shift)).astype(np.float32)
    qs[20:] += np.float32(0.375)  # half the queries fractional
    oidx = oracle.build_index(base, 4, 10, 3, 42, 0)
    idx = gpu.load_index(oidx.serialize(), base)
    for a, b, k in ((0.05, 0.01, 10), (0.05, 0.02, 40), (0.2, 0.05, 1)):
        ids, dd = idx.knn_query_batch(qs, gpu.CollisionParams(a, b, k))
        oi, od, _ = oidx.knn_query_batch(base, qs, a, b, k)
        assert np.array_equal(ids, oi), (d, shift, a, b, k)
        assert np.array_equal(dd, od), (d, shift, a, b, k)


@pytest.mark.parametrize("fused", ["1", "0", "stage"])
@pytest.mark.parametrize("words", ["1", "2"])
def test_dense_select_block_widths(gpu, oracle, words, fused, monkeypatch):
    """32-query (one mask word) and 64-query (two words) dense blocks, single-pass (with its
    fallback; direct or staged buffer stores) and two-pass, give the same candidate sets and answers as the reference; a partial
    last block (nq % 64 != 0) included."""
    monkeypatch.setenv("SUCO_DENSE_WORDS", words)
    monkeypatch.setenv("SUCO_DENSE_FUSED", "0" if fused == "0" else "1")
    if fused == "stage":  # the fused pass's staged (8-byte) buffer stores, normally for dense supersets
        monkeypatch.setenv("SUCO_DENSE_STAGE", "1")
    full = oracle.clustered(60000 + 77, 24, 30, 2024, 0, 100, 9, True)  # 30 pieces: a real sample
    base, qs = oracle.hold_out(full, 77, 2025)
    oidx = oracle.build_index(base, 6, 20, 3, 42, 0)
    idx = gpu.load_index(oidx.serialize(), base)
    for a, b, k in ((0.05, 0.01, 10), (0.01, 0.2, 33)):
        ids, dd = idx.knn_query_batch(qs, gpu.CollisionParams(a, b, k))
        oi, od, _ = oidx.knn_query_batch(base, qs, a, b, k)
        assert np.array_equal(ids, oi) and np.array_equal(dd, od), (words, a, b, k)
    s1, c1, _, _ = idx.query_intermediates(qs[5], gpu.CollisionParams(0.05, 0.01, 10))
    s2, c2, _, _ = oidx.query_intermediates(base, qs[5], 0.05, 0.01, 10)
    assert np.array_equal(c1, c2)


@pytest.mark.parametrize("overlap", ["0", "1"])
def test_dense_buffer_overflow_falls_back(gpu, oracle, overlap, monkeypatch, capfd):
    """Rows sorted along one coordinate put a query's high scorers in a few neighbouring pieces:
    more than B = 96 of them in one (query, piece) buffer flags the query, which then takes the exact
    two-pass select. Answers stay identical to the reference — with the fallback on the select
    stream, and overlapped with the re-rank of the unflagged queries (re-ranked in a second pass over
    the flagged list; k > 32 takes the generic top-k kernel through the same mapping)."""
    monkeypatch.setenv("SUCO_FB_OVERLAP", overlap)
    monkeypatch.setenv("SUCO_DENSE_STATS", "1")
    monkeypatch.setenv("SUCO_DENSE_BUF", "96")  # small batches would otherwise get whole-piece buffers
    full = oracle.clustered(40000 + 64, 16, 8, 77, 0, 100, 6, True)
    full = full[np.argsort(full[:, 0], kind="stable")]
    rng = np.random.default_rng(5)
    pick = np.sort(rng.choice(len(full), 64, replace=False))
    qs = full[pick]
    base = np.delete(full, pick, axis=0)
    oidx = oracle.build_index(base, 4, 12, 3, 42, 0)
    idx = gpu.load_index(oidx.serialize(), base)
    for a, b, k in ((0.2, 0.01, 10), (0.05, 0.02, 20), (0.05, 0.02, 40)):
        ids, dd = idx.knn_query_batch(qs, gpu.CollisionParams(a, b, k))
        oi, od, _ = oidx.knn_query_batch(base, qs, a, b, k)
        assert np.array_equal(ids, oi) and np.array_equal(dd, od), (a, b, k)
        fi, fd = idx.knn_query_batch(qs.astype(np.float32) + np.float32(0.25), gpu.CollisionParams(a, b, k))
        gi, gd, _ = oidx.knn_query_batch(base, qs.astype(np.float32) + np.float32(0.25), a, b, k)
        assert np.array_equal(fi, gi) and np.array_equal(fd, gd), ("non-integer queries", a, b, k)
    err = capfd.readouterr().err
    flagged = [int(line.split("dense select: ")[1].split(" of")[0]) for line in err.splitlines()
               if "dense select:" in line]
    assert flagged and max(flagged) > 0, err


@pytest.mark.parametrize("fused", ["1", "0", "pair"])
@pytest.mark.parametrize("ns,kh,nq", [(6, 20, 77), (8, 30, 40), (3, 45, 16)])
def test_dense_half_width_mode(gpu, oracle, ns, kh, fused, nq, monkeypatch):
    """The half-width dense select (16-query blocks, u16 masks, two points per lane — the mode config
    5's 8 x 10,000 cells take) forced on small tables: single-pass and two-pass, N_s < 8 (code
    positions past N_s), a partial last query block and a partial last 64-point tile; "pair": the
    single pass on 2-CTA clusters (32-bit masks of 4 subspaces per CTA, DSMEM exchange; N_s >= 5)."""
    monkeypatch.setenv("SUCO_DENSE_HALF", "2")
    monkeypatch.setenv("SUCO_DENSE_FUSED", "0" if fused == "0" else "1")
    monkeypatch.setenv("SUCO_DENSE_PAIR", "1" if fused == "pair" else "0")
    full = oracle.clustered(60000 + nq, 24, 30, 2024 + ns, 0, 100, 9, True)
    base, qs = oracle.hold_out(full, nq, 2025)
    oidx = oracle.build_index(base, ns, kh, 3, 42, 0)
    idx = gpu.load_index(oidx.serialize(), base)
    for a, b, k in ((0.05, 0.01, 10), (0.01, 0.2, 33), (0.3, 0.002, 5)):
        ids, dd = idx.knn_query_batch(qs, gpu.CollisionParams(a, b, k))
        oi, od, _ = oidx.knn_query_batch(base, qs, a, b, k)
        assert np.array_equal(ids, oi) and np.array_equal(dd, od), (ns, a, b, k)
    s1, c1, _, _ = idx.query_intermediates(qs[3], gpu.CollisionParams(0.05, 0.01, 10))
    s2, c2, _, _ = oidx.query_intermediates(base, qs[3], 0.05, 0.01, 10)
    assert np.array_equal(c1, c2)


def test_dense_half_width_overflow_falls_back(gpu, oracle, monkeypatch, capfd):
    """Half-width mode: an overflowing (query, piece) buffer flags its query for the exact two-pass
    select (as test_dense_buffer_overflow_falls_back)."""
    monkeypatch.setenv("SUCO_DENSE_HALF", "2")
    monkeypatch.setenv("SUCO_DENSE_STATS", "1")
    monkeypatch.setenv("SUCO_DENSE_BUF", "96")
    full = oracle.clustered(40000 + 40, 16, 8, 77, 0, 100, 6, True)
    full = full[np.argsort(full[:, 0], kind="stable")]
    pick = np.sort(np.random.default_rng(5).choice(len(full), 40, replace=False))
    qs, base = full[pick], np.delete(full, pick, axis=0)
    oidx = oracle.build_index(base, 4, 12, 3, 42, 0)
    idx = gpu.load_index(oidx.serialize(), base)
    for a, b, k in ((0.2, 0.01, 10), (0.05, 0.02, 20), (0.05, 0.02, 40)):
        ids, dd = idx.knn_query_batch(qs, gpu.CollisionParams(a, b, k))
        oi, od, _ = oidx.knn_query_batch(base, qs, a, b, k)
        assert np.array_equal(ids, oi) and np.array_equal(dd, od), (a, b, k)
        fi, fd = idx.knn_query_batch(qs.astype(np.float32) + np.float32(0.25), gpu.CollisionParams(a, b, k))
        gi, gd, _ = oidx.knn_query_batch(base, qs.astype(np.float32) + np.float32(0.25), a, b, k)
        assert np.array_equal(fi, gi) and np.array_equal(fd, gd), ("non-integer queries", a, b, k)
    err = capfd.readouterr().err
    flagged = [int(line.split("dense select: ")[1].split(" of")[0]) for line in err.splitlines()
               if "dense select:" in line]
    assert flagged and max(flagged) > 0, err


@pytest.mark.parametrize("dups", [40, 3000])
def test_screened_rerank_ties(gpu, oracle, ref, dups):
    """The fp32-screened re-rank (float rows, k <= 32) with masses of exact distance ties: `dups`
    copies of one row next to the queries. 3000 copies overflow the per-warp buffers of rows that
    pass the screen, so those queries are re-ranked exactly from scratch; answers stay identical
    to the reference either way (ids by (distance, id))."""
    full = oracle.clustered(8000 + 12, 32, 10, 99, 0, 1, 0.05, False)
    base, qs = oracle.hold_out(full, 12, 100)
    base = np.concatenate([base, np.repeat(base[17:18], dups, axis=0)])
    qs = np.concatenate([qs, base[17:18] + np.float32(1e-3), base[17:18]])
    oidx = oracle.build_index(base, 4, 10, 3, 42, 0)
    idx = gpu.load_index(oidx.serialize(), base)
    # k > 32: the radix top-k; 3000 equal distances overflow its bucket into the k-round kernel
    for a, b, k in ((1.0, 1.0, 10), (0.3, 0.2, 32), (0.05, 0.01, 1), (0.3, 0.2, 64), (1.0, 1.0, 200)):
        ids, dd = idx.knn_query_batch(qs, gpu.CollisionParams(a, b, k))
        oi, od, _ = oidx.knn_query_batch(base, qs, a, b, k)
        assert np.array_equal(ids, oi) and np.array_equal(dd, od), (dups, a, b, k)
    ids, dd = idx.exact_knn_batch(qs, 10)
    for i, q in enumerate(qs):
        wi, wd = ref.exact_knn(base, q, 10)
        assert np.array_equal(ids[i], wi) and np.array_equal(dd[i], wd), (dups, i)


@pytest.mark.parametrize("scale", [1e-22, 1e20])
def test_screened_rerank_extreme_magnitudes(gpu, oracle, scale):
    """Float rows whose squared distances underflow (1e-22) or overflow (1e20) fp32: the screen's
    absolute slack and its 'non-finite always passes' rule keep the answers exact."""
    full = oracle.clustered(3000 + 8, 16, 6, 7, 0, 1, 0.1, False) * np.float32(scale)
    base, qs = oracle.hold_out(full, 8, 8)
    oidx = oracle.build_index(base, 2, 6, 2, 42, 0)
    idx = gpu.load_index(oidx.serialize(), base)
    for a, b, k in ((1.0, 1.0, 10), (0.2, 0.05, 5)):
        ids, dd = idx.knn_query_batch(qs, gpu.CollisionParams(a, b, k))
        oi, od, _ = oidx.knn_query_batch(base, qs, a, b, k)
        assert np.array_equal(ids, oi) and np.array_equal(dd, od), (scale, a, b, k)


@pytest.mark.parametrize("prefix", ["0", "1", "3"])
def test_int8_screen_forced(gpu, oracle, ref, prefix, monkeypatch):
    """The int8-screened re-rank (SUCO_Q8=2: even for short candidate lists) with plain records
    (prefix 0) and the prefix-bound layouts of 16 and 48 dims: masses of exact ties next to the
    queries, squared distances that underflow / overflow fp32, and the float / 8 x 64^2-cell
    corpora of test_knn_vs_oracle — answers identical to the reference."""
    monkeypatch.setenv("SUCO_Q8", "2")
    monkeypatch.setenv("SUCO_Q8_PREFIX", prefix)
    full = oracle.clustered(8000 + 12, 64, 10, 99, 0, 1, 0.05, False)
    base, qs = oracle.hold_out(full, 12, 100)
    base = np.concatenate([base, np.repeat(base[17:18], 3000, axis=0)])
    qs = np.concatenate([qs, base[17:18] + np.float32(1e-3), base[17:18]])
    oidx = oracle.build_index(base, 4, 10, 3, 42, 0)
    idx = gpu.load_index(oidx.serialize(), base)
    for a, b, k in ((1.0, 1.0, 10), (0.3, 0.2, 32), (0.05, 0.01, 1), (0.3, 0.2, 64)):
        ids, dd = idx.knn_query_batch(qs, gpu.CollisionParams(a, b, k))
        oi, od, _ = oidx.knn_query_batch(base, qs, a, b, k)
        assert np.array_equal(ids, oi) and np.array_equal(dd, od), (prefix, a, b, k)
    for scale in (1e-22, 1e20):
        full = oracle.clustered(3000 + 8, 96, 6, 7, 0, 1, 0.1, False) * np.float32(scale)
        base2, qs2 = oracle.hold_out(full, 8, 8)
        oidx2 = oracle.build_index(base2, 2, 6, 2, 42, 0)
        idx2 = gpu.load_index(oidx2.serialize(), base2)
        for a, b, k in ((1.0, 1.0, 10), (0.2, 0.05, 5)):
            ids, dd = idx2.knn_query_batch(qs2, gpu.CollisionParams(a, b, k))
            oi, od, _ = oidx2.knn_query_batch(base2, qs2, a, b, k)
            assert np.array_equal(ids, oi) and np.array_equal(dd, od), (prefix, scale, a, b, k)
    if prefix == "3":  # wide rows (128 < d <= 1024): the prefix screen's warp-cooperative second stage
        for d in (140, 384):
            full = oracle.clustered(4000 + 10, d, 8, 5 + d, 0, 1, 0.05, False)
            base4, qs4 = oracle.hold_out(full, 10, 77)
            base4 = np.concatenate([base4, np.repeat(base4[3:4], 500, axis=0)])
            qs4 = np.concatenate([qs4, base4[3:4]])
            oidx4 = oracle.build_index(base4, 4, 8, 2, 42, 0)
            idx4 = gpu.load_index(oidx4.serialize(), base4)
            for a, b, k in ((1.0, 1.0, 10), (0.3, 0.2, 32), (0.2, 0.05, 5)):
                ids, dd = idx4.knn_query_batch(qs4, gpu.CollisionParams(a, b, k))
                oi, od, _ = oidx4.knn_query_batch(base4, qs4, a, b, k)
                assert np.array_equal(ids, oi) and np.array_equal(dd, od), (prefix, d, a, b, k)
    for case in ("float", "dense_1024"):
        n, d, cl, lo, hi, sig, quant, ns, kh, it, mode, plist = CASES[case]
        full = oracle.clustered(n + 40, d, cl, 1000 + n, lo, hi, sig, quant)
        base3, qs3 = oracle.hold_out(full, 40, 1001 + n)
        oidx3 = oracle.build_index(base3, ns, kh, it, 42, mode)
        idx3 = gpu.load_index(oidx3.serialize(), base3)
        for a, b, k in plist:
            ids, dd = idx3.knn_query_batch(qs3, gpu.CollisionParams(a, b, k))
            oi, od, _ = oidx3.knn_query_batch(base3, qs3, a, b, k)
            assert np.array_equal(ids, oi) and np.array_equal(dd, od), (prefix, case, a, b, k)


@pytest.mark.parametrize("fused", ["1", "0"])
@pytest.mark.parametrize("ns,kh", [(16, 12), (12, 20), (9, 7)])
def test_dense_select_16_subspaces(gpu, oracle, ns, kh, fused, monkeypatch):
    """9..16 subspaces (config 3 has 16): two code vectors per point, five score planes and 16
    histogram levels in the dense select, single-pass and two-pass; partial last query block."""
    monkeypatch.setenv("SUCO_DENSE_FUSED", fused)
    d = 4 * ns
    full = oracle.clustered(50000 + 45, d, 30, 3030 + ns, 0, 100, 9, False)
    base, qs = oracle.hold_out(full, 45, 3031)
    oidx = oracle.build_index(base, ns, kh, 3, 42, 0)
    idx = gpu.load_index(oidx.serialize(), base)
    for a, b, k in ((0.05, 0.01, 10), (0.3, 0.002, 7), (0.01, 0.2, 20)):
        ids, dd = idx.knn_query_batch(qs, gpu.CollisionParams(a, b, k))
        oi, od, _ = oidx.knn_query_batch(base, qs, a, b, k)
        assert np.array_equal(ids, oi) and np.array_equal(dd, od), (ns, a, b, k)
    s1, c1, _, _ = idx.query_intermediates(qs[4], gpu.CollisionParams(0.05, 0.01, 10))
    s2, c2, _, _ = oidx.query_intermediates(base, qs[4], 0.05, 0.01, 10)
    assert np.array_equal(c1, c2)


@pytest.mark.parametrize("nocut", ["0", "1"])
def test_dense_tie_cut_sorted_corpus(gpu, oracle, monkeypatch, capfd, nocut):
    """The single pass stores score == L entries only in the pieces the tie quota is expected to
    reach. Rows sorted along one coordinate concentrate a query's ties in a few pieces, so the
    estimate misses for some queries, which take the exact fallback; answers are identical to the
    reference with and without the cut."""
    monkeypatch.setenv("SUCO_DENSE_STATS", "1")
    if nocut == "1":
        monkeypatch.setenv("SUCO_DENSE_NOCUT", "1")
    full = oracle.clustered(120000 + 64, 16, 8, 78, 0, 100, 6, True)
    full = full[np.argsort(-full[:, 0], kind="stable")]
    pick = np.sort(np.random.default_rng(6).choice(len(full), 64, replace=False))
    qs, base = full[pick], np.delete(full, pick, axis=0)
    oidx = oracle.build_index(base, 4, 12, 3, 42, 0)
    idx = gpu.load_index(oidx.serialize(), base)
    for a, b, k in ((0.2, 0.01, 10), (0.05, 0.02, 20), (0.5, 0.001, 5)):
        ids, dd = idx.knn_query_batch(qs, gpu.CollisionParams(a, b, k))
        oi, od, _ = oidx.knn_query_batch(base, qs, a, b, k)
        assert np.array_equal(ids, oi) and np.array_equal(dd, od), (a, b, k)


def test_host_batch_chunked_io(gpu, oracle):
    """Host-buffer calls of >= 2048 queries upload queries and download results in chunks that
    overlap the traversal and re-rank of their neighbours; answers equal the reference's, including
    a ragged last chunk, k > 32 and k = 1."""
    full = oracle.clustered(8000 + 2503, 24, 20, 4242, 0, 100, 8, True)
    base, qs = oracle.hold_out(full, 2503, 4243)
    oidx = oracle.build_index(base, 4, 10, 3, 42, 0)
    idx = gpu.load_index(oidx.serialize(), base)
    for a, b, k in ((0.05, 0.01, 10), (0.2, 0.05, 40), (0.1, 0.002, 1)):
        ids, dd = idx.knn_query_batch(qs, gpu.CollisionParams(a, b, k))
        oi, od, _ = oidx.knn_query_batch(base, qs, a, b, k)
        assert np.array_equal(ids, oi) and np.array_equal(dd, od), (a, b, k)


def test_concurrent_queries_one_index(gpu, oracle):
    """The index is immutable (index.hpp:63-66): four host threads query one index at once — two
    with their own query contexts (the reference's QueryScratch, query.hpp:72-78), two through the
    index's context pool — each on a different parameter set, all equal to the oracle."""
    import threading
    full = oracle.clustered(30000 + 300, 24, 20, 909, 0, 100, 8, True)
    base, qs = oracle.hold_out(full, 300, 910)
    oidx = oracle.build_index(base, 4, 12, 3, 42, 0)
    idx = gpu.load_index(oidx.serialize(), base)
    plist = [(0.05, 0.01, 10), (0.1, 0.005, 40), (0.02, 0.02, 5), (0.2, 0.002, 1)]
    want = [oidx.knn_query_batch(base, qs, a, b, k)[:2] for a, b, k in plist]
    ctxs = [idx.context(), idx.context(), None, None]
    got, errs = [None] * 4, []

    def run(t):
        try:
            for _ in range(3):
                got[t] = idx.knn_query_batch(qs, gpu.CollisionParams(*plist[t]), scratch=ctxs[t])
        except Exception as e:  # noqa: BLE001
            errs.append(e)
    ts = [threading.Thread(target=run, args=(t,)) for t in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for t in range(4):
        assert np.array_equal(got[t][0], want[t][0]) and np.array_equal(got[t][1], want[t][1]), plist[t]


@pytest.mark.parametrize("overlap", ["0", "1"])
@pytest.mark.parametrize("knob", ["tiles", "scratch"])
def test_multi_tile_pipeline(gpu, oracle, knob, overlap, monkeypatch):
    """Batches split into several pipeline tiles (SUCO_TILES, or a small SUCO_SCRATCH_MB budget):
    slot reuse across tiles and the cross-stream events — the overlapped dense fallback included —
    keep every answer equal to the oracle."""
    if knob == "tiles":
        monkeypatch.setenv("SUCO_TILES", "3")
    else:
        monkeypatch.setenv("SUCO_SCRATCH_MB", "24")
    monkeypatch.setenv("SUCO_FB_OVERLAP", overlap)
    monkeypatch.setenv("SUCO_DENSE_BUF", "96")
    full = oracle.clustered(40000 + 700, 16, 8, 77, 0, 100, 6, True)
    full = full[np.argsort(full[:, 0], kind="stable")]  # clustered ids: some queries take the fallback
    pick = np.sort(np.random.default_rng(9).choice(len(full), 700, replace=False))
    qs, base = full[pick], np.delete(full, pick, axis=0)
    oidx = oracle.build_index(base, 4, 12, 3, 42, 0)
    idx = gpu.load_index(oidx.serialize(), base)
    ctx = idx.context()
    for a, b, k in ((0.2, 0.01, 10), (0.05, 0.02, 40)):
        ids, dd = idx.knn_query_batch(qs, gpu.CollisionParams(a, b, k), scratch=ctx)
        oi, od, _ = oidx.knn_query_batch(base, qs, a, b, k)
        assert np.array_equal(ids, oi) and np.array_equal(dd, od), (knob, a, b, k)
    assert ctx.last_launches() > 20  # several tiles' kernels


def test_null_buffers_are_contract_errors(gpu):
    """Every query entry point rejects NULL buffers for nq > 0 (CONTRACT), after the reference's
    own checks."""
    import ctypes as C
    from paper_2411_14754_b200 import _capi
    g = golden("e2e_small.npz")
    idx = gpu.load_index(g["index"].tobytes(), g["base"])
    cp = gpu.CollisionParams(0.05, 0.05, 10)._c()
    q = np.ascontiguousarray(g["queries"][:2])
    ids = np.zeros((2, 10), np.uint32)
    dd = np.zeros((2, 10), np.float64)
    qp, ip, dp = (a.ctypes.data_as(t) for a, t in ((q, _capi.f32p), (ids, _capi.u32p), (dd, _capi.f64p)))
    for args in ((None, ip, dp), (qp, None, dp), (qp, ip, None)):
        assert _capi.knn_query_batch(idx.handle, args[0], 2, q.shape[1], C.byref(cp), args[1], args[2], None) == 5
    assert _capi.knn_query_batch_device(idx.handle, None, 2, q.shape[1], C.byref(cp), None, None, None, None) == 5
    assert _capi.knn_query_batch(idx.handle, None, 0, q.shape[1], C.byref(cp), None, None, None) == 0
