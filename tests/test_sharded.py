"""Multi-GPU shard protocol.

CPU: the protocol model (tests/shard_protocol_model.py — the library's three
exchange rounds restated) in one process for G = 1..5 and over gloo with
world_size 2, against the unsharded oracle.
GPU: the library's own sharded query and sharded build over the in-process
communicator (G ranks on G threads, all on cuda:0 — each collective meets at
a host barrier, so no kernel waits on another rank), bit-identical to the
oracle for G = 1..8.
"""
import os
import socket

import numpy as np
import pytest

from conftest import ROOT

PARAMS = ((0.05, 0.02, 10), (0.1, 0.005, 7), (0.002, 0.3, 12))  # the last: T = 0, zero-score ties


def _corpus(oracle, n=3000, d=16, seed=5, nq=12):
    full = oracle.clustered(n + nq, d, 10, seed, 0.0, 60.0, 5.0, True)
    return oracle.hold_out(full, nq, seed + 1)


class _P:
    def __init__(self, a, b, k):
        self.alpha, self.beta, self.k = a, b, k


def _m(b, n, k):
    import math
    x = b * n
    x = round(x) if abs(x - round(x)) <= 1e-6 else x
    return max(k, math.ceil(x))


@pytest.mark.parametrize("G,block,piece", [(1, 256, 64), (2, 128, 32), (3, 96, 32), (5, 64, 64)])
def test_model_inprocess_matches_unsharded(oracle, G, block, piece):
    from shard_protocol_model import ModelShard, run_inprocess
    base, qs = _corpus(oracle)
    oidx = oracle.build_index(base, 4, 8, 3, 42, 0)
    shards = [ModelShard(oracle, oidx, base, r, G, block, piece) for r in range(G)]
    for a, b, k in PARAMS:
        wi, wd, _ = oidx.knn_query_batch(base, qs, a, b, k)
        for ids, dd in run_inprocess(shards, qs, _P(a, b, k), _m(b, len(base), k)):
            assert np.array_equal(ids, wi), (G, a, b, k)
            assert np.array_equal(dd, wd), (G, a, b, k)


def _worker(rank, world, port, q):
    try:
        import sys
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        sys.path.insert(0, ROOT)
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from oracle.oracle import oracle
        from shard_protocol_model import ModelShard, torch_allgather
        O = oracle()
        base, qs = _corpus(O)
        oidx = O.build_index(base, 4, 8, 3, 42, 0)
        sh = ModelShard(O, oidx, base, rank, world, 128, 32)
        out = [sh.query(qs, _P(a, b, k), _m(b, len(base), k), torch_allgather) for a, b, k in PARAMS]
        q.put((rank, out))
        dist.destroy_process_group()
    except Exception:  # surface worker failures to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


def test_gloo_world_size_2_matches_unsharded(oracle):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in (0, 1):
        assert not isinstance(res[r], str), res[r]
    base, qs = _corpus(oracle)
    oidx = oracle.build_index(base, 4, 8, 3, 42, 0)
    for i, (a, b, k) in enumerate(PARAMS):
        wi, wd, _ = oidx.knn_query_batch(base, qs, a, b, k)
        for r in (0, 1):
            ids, dd = res[r][i]
            assert np.array_equal(ids, wi), (r, a, b, k)
            assert np.array_equal(dd, wd), (r, a, b, k)


def test_block_hint(suco):
    from paper_2411_14754_b200.sharded import block_hint, shard_ids
    assert block_hint(10_000_000, 8) == 8192      # cfg4
    assert block_hint(100_000_000, 8) == 65536    # cfg5
    assert block_hint(20_000, 4) == 2048          # floor: one dense piece
    ids = [shard_ids(10_000, 2048, 3, r) for r in range(3)]
    assert np.array_equal(np.sort(np.concatenate(ids)), np.arange(10_000))
    assert ids[1][0] == 2048 and ids[0][2048] == 3 * 2048


# ------------------------------------------------------------------ GPU
GPU_PARAMS = ((0.05, 0.005, 10), (0.02, 0.05, 40), (0.3, 0.001, 3), (0.001, 0.4, 5))


def _gpu_corpus(oracle, G, n=20000, d=32, nq=50, quant=True):
    if quant:
        full = oracle.clustered(n + nq, d, 40, 77 + G, 20, 140, 18, True)
    else:
        full = oracle.clustered(n + nq, d, 40, 77 + G, 0.0, 1.0, 0.05, False)
    return oracle.hold_out(full, nq, 78)


@pytest.mark.gpu
@pytest.mark.parametrize("G,block", [(1, 4096), (2, 2048), (3, 2048), (4, 4096), (5, 2048), (8, 2048), (3, 6144)])
def test_gpu_sharded_query_matches_oracle(gpu, oracle, G, block):
    """The library's sharded query (three device all-gathers, G-way merge) on G shards cut from one
    index, every rank's answer against the unsharded ORACLE; the last parameter set has fewer than
    m colliding points (T = 0: the quota is filled with the lowest-id zero scorers)."""
    from paper_2411_14754_b200.sharded import Shard, emulate
    base, qs = _gpu_corpus(oracle, G)
    oidx = oracle.build_index(base, 4, 16, 3, 42, 0)
    idx = gpu.load_index(oidx.serialize(), base)
    shards = [Shard.cut(idx, r, G, block) for r in range(G)]
    for a, b, k in GPU_PARAMS:
        want_i, want_d, _ = oidx.knn_query_batch(base, qs, a, b, k)
        for r, (ids, dd) in enumerate(emulate(shards, qs, gpu.CollisionParams(a, b, k))):
            assert np.array_equal(ids, want_i), (G, block, r, a, b, k)
            assert np.array_equal(dd, want_d), (G, block, r, a, b, k)


@pytest.mark.gpu
@pytest.mark.parametrize("G", [2, 4])
def test_gpu_sharded_query_float_rows_and_half_mode(gpu, oracle, G, monkeypatch):
    """Float rows (the fp32-screened re-rank), a shuffled layout, and the half-width dense select
    (config 5's mode) on the shards."""
    from paper_2411_14754_b200.sharded import Shard, emulate
    monkeypatch.setenv("SUCO_DENSE_HALF", "2")
    base, qs = _gpu_corpus(oracle, G, n=16000, d=24, nq=30, quant=False)
    oidx = oracle.build_index(base, 3, 10, 3, 1, 1)
    idx = gpu.load_index(oidx.serialize(), base)
    shards = [Shard.cut(idx, r, G, 2048) for r in range(G)]
    for a, b, k in ((0.05, 0.01, 10), (0.2, 0.002, 33)):
        want_i, want_d, _ = oidx.knn_query_batch(base, qs, a, b, k)
        for ids, dd in emulate(shards, qs, gpu.CollisionParams(a, b, k)):
            assert np.array_equal(ids, want_i) and np.array_equal(dd, want_d), (G, a, b, k)


@pytest.mark.gpu
@pytest.mark.parametrize("G", [1, 2, 3, 8])
@pytest.mark.parametrize("sampled", [False, True])
def test_gpu_sharded_build_equals_cut_of_full_build(gpu, oracle, G, sampled):
    """suco_gpu_build_shard (k-means jobs spread over the ranks, centroids broadcast, local rows
    assigned, cell counts all-reduced), each rank given only its own rows: every shard equals the
    same shard cut from the single-GPU build — centroids, local IMI — and answers like the oracle."""
    from paper_2411_14754_b200.sharded import Comm, Shard, run_ranks, shard_ids
    n, block = 24000, 2048
    full = oracle.clustered(n + 40, 24, 30, 500 + G, 0, 100, 8, True)
    base, qs = oracle.hold_out(full, 40, 501)
    params = gpu.IndexParams(4, 12, 3, 42)
    train = np.sort(np.random.default_rng(G).choice(n, 3000, replace=False)).astype(np.uint32) if sampled else None
    whole = gpu.build_index_sampled(base, train, params) if sampled else gpu.build_index(base, params)
    comms = Comm.local(G)
    built = run_ranks(lambda r: Shard.build(base[shard_ids(n, block, G, r)], n, params, block, comms[r],
                                            train_ids=train), G)
    for r in range(G):
        cut = Shard.cut(whole, r, G, block)
        assert built[r].shard_info() == cut.shard_info()
        for s in range(params.num_subspaces):
            a, b = built[r].subspace(s), cut.subspace(s)
            for x, y in zip(a[:2], b[:2]):
                assert np.array_equal(x, y), (G, r, s, "centroids")
            nl = cut.shard_info()["n_local"]
            assert np.array_equal(a[2], b[2]) and np.array_equal(a[3][:nl], b[3][:nl]), (G, r, s, "IMI")
    blob = whole.serialize()
    oidx = oracle.load_index(blob)
    cp = (0.05, 0.01, 10)
    want_i, want_d, _ = oidx.knn_query_batch(base, qs, *cp)
    outs = run_ranks(lambda r: built[r].knn_query_batch(comms[r], qs, gpu.CollisionParams(*cp)), G)
    for ids, dd in outs:
        assert np.array_equal(ids, want_i) and np.array_equal(dd, want_d), (G, sampled)
    for c in comms:
        c.close()


@pytest.mark.gpu
def test_gpu_sharded_build_error_reaches_every_rank(gpu):
    """A non-finite value in one rank's rows fails the build on every rank (no rank left blocked)."""
    from paper_2411_14754_b200.sharded import Comm, Shard, run_ranks, shard_ids
    n, block, G = 8192, 2048, 2
    base = np.random.default_rng(1).integers(0, 50, size=(n, 8)).astype(np.float32)
    base[5000, 3] = np.inf  # block 2: rank 0
    comms = Comm.local(G)
    errs = []

    def one(r):
        try:
            Shard.build(base[shard_ids(n, block, G, r)], n, gpu.IndexParams(2, 4, 2, 42), block, comms[r])
        except gpu.Error as e:
            errs.append((r, type(e).__name__))
    run_ranks(one, G)
    assert sorted(errs) == [(0, "ContractError"), (1, "ContractError")]


@pytest.mark.gpu
def test_gpu_shard_exchange_volume(gpu, oracle, monkeypatch):
    """Bytes each rank sends per query. Two-pass protocol: 64 (totals) + 4 x ceil(#blocks / G)
    (tie counts) + 12 k (local top-k). Single pass: 68 (sampled totals) + 4 (#(score > L)) +
    4 x ceil(#blocks / G) + 12 k, plus 4 per tile (the flag count); a tile some shard flagged also
    runs the two-pass exchange. Never the per-piece histograms."""
    from paper_2411_14754_b200.sharded import Comm, Shard, run_ranks
    base, qs = _gpu_corpus(oracle, 4)
    G, block = 4, 2048
    nb = -(-len(base) // block)
    nblm = -(-nb // G)
    cp = gpu.CollisionParams(0.05, 0.005, 10)
    nq = len(qs)
    two = 64 + 4 * nblm
    one = 68 + 4 + 4 * nblm
    for fused in ("0", "1"):
        monkeypatch.setenv("SUCO_DENSE_FUSED", fused)
        idx = gpu.build_index(base, gpu.IndexParams(4, 16, 3, 42))
        shards = [Shard.cut(idx, r, G, block) for r in range(G)]
        ctxs = [s.context() for s in shards]
        comms = Comm.local(G)
        run_ranks(lambda r: shards[r].knn_query_batch(comms[r], qs, cp, scratch=ctxs[r]), G)
        got = [c.exchange_bytes() for c in ctxs]
        if fused == "0":
            want = {nq * (two + 12 * cp.k)}
        else:
            want = {nq * (one + 12 * cp.k) + 4, nq * (one + two + 12 * cp.k) + 4}
        assert all(v in want for v in got), (fused, got, want)
        for c in comms:
            c.close()


@pytest.mark.gpu
def test_gpu_shard_errors(gpu, oracle):
    from paper_2411_14754_b200.sharded import Comm, Shard
    base, qs = _gpu_corpus(oracle, 2)
    idx = gpu.build_index(base, gpu.IndexParams(4, 16, 3, 42))
    with pytest.raises(gpu.ConfigError):
        Shard.cut(idx, 0, 2, 1000)  # not a multiple of 2048
    with pytest.raises(gpu.ConfigError):
        Shard.cut(idx, 2, 2, 2048)
    sh = Shard.cut(idx, 1, 2, 2048)
    comms = Comm.local(2)
    with pytest.raises(gpu.ContractError):  # rank 0's member does not hold shard 1
        sh.knn_query_batch(comms[0], qs, gpu.CollisionParams())
    with pytest.raises(gpu.ContractError):
        idx.knn_query_batch(qs, gpu.CollisionParams(), scratch=sh.context())  # another index's context
    with pytest.raises(gpu.ContractError):
        sh.serialize()
