"""Multi-GPU shard protocol: exchange math, gloo world_size-2 run on CPU, and
single-GPU emulation of G shards — all bit-identical to the unsharded results."""
import os
import socket

import numpy as np
import pytest
import torch

from conftest import ROOT


def _corpus(oracle, n=1500, d=16, seed=5):
    full = oracle.clustered(n + 12, d, 10, seed, 0.0, 60.0, 5.0, True)
    return oracle.hold_out(full, 12, seed + 1)


@pytest.mark.parametrize("ppb", [1, 3])
def test_plan_matches_reference_selection_rule(ppb):
    """T and id-ordered quotas from per-piece histograms == top-m by (score desc, id asc); pieces
    are whole blocks (ppb = 1) or ppb consecutive sub-pieces of each block (dense select)."""
    from paper_2411_14754_b200.sharded import plan_for_shard
    rng = np.random.default_rng(ppb)
    ns, n, ps, G, m = 6, 997, 13, 3, 61
    b = ps * ppb
    for _ in range(20):
        scores = rng.integers(0, ns + 1, size=n)
        order = sorted(range(n), key=lambda i: (-scores[i], i))
        want = set(order[:m])
        nb = -(-n // b)

        def pieces_of(r):  # (global start, end) of shard r's pieces in local order
            out = []
            for j in (j for j in range(nb) if j % G == r):
                for sub in range(ppb):
                    lo = j * b + sub * ps
                    if lo < n:
                        out.append((lo, min(n, lo + ps, (j + 1) * b)))
            return out
        hists = []
        for r in range(G):
            pcs = pieces_of(r)
            h = np.zeros((1, len(pcs), ns + 2), np.int32)
            for pi, (lo, hi) in enumerate(pcs):
                for t in range(ns + 1):
                    h[0, pi, t] = (scores[lo:hi] >= t).sum()
            hists.append(torch.from_numpy(h))
        got = set()
        for r in range(G):
            plan = plan_for_shard(hists, r, m, ppb)
            T = int(plan.T[0])
            mine = set()
            for pi, (lo, hi) in enumerate(pieces_of(r)):
                s = scores[lo:hi]
                mine |= set((np.nonzero(s > T)[0] + lo).tolist())
                mine |= set((np.nonzero(s == T)[0] + lo)[: int(plan.quota[0, pi])].tolist())
            assert int(plan.counts[0]) == len(mine)
            got |= mine
        assert got == want


def _worker(rank, world, port, q, split=False):
    try:
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import sys
        sys.path.insert(0, ROOT)
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from oracle.oracle import oracle
        from shard_oracle_engine import OracleShard, OracleSplitShard
        from paper_2411_14754_b200 import CollisionParams
        from paper_2411_14754_b200.sharded import TorchComm, knn_query_distributed
        O = oracle()
        base, qs = _corpus(O)
        oidx = O.build_index(base, 4, 8, 3, 42, 0)
        eng = (OracleSplitShard if split else OracleShard)(O, oidx, base, rank, world, 64)
        eng._queries = torch.from_numpy(qs)
        comm = TorchComm()
        out = []
        for a, bta, k in ((0.05, 0.02, 10), (0.1, 0.005, 7), (0.002, 0.3, 12)):
            ids, dd = knn_query_distributed(eng, comm, torch.from_numpy(qs), CollisionParams(a, bta, k))
            out.append((ids.numpy(), dd.numpy()))
        q.put((rank, out))
        dist.destroy_process_group()
    except Exception as e:  # surface worker failures to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("split", [False, True])
def test_gloo_world_size_2_matches_unsharded(oracle, split):
    """Both protocols over gloo: replicated traversal, and the query-split traversal whose cell
    lists are all-gathered (split=True)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, split)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in (0, 1):
        assert not isinstance(res[r], str), res[r]
    base, qs = _corpus(oracle)
    oidx = oracle.build_index(base, 4, 8, 3, 42, 0)
    for i, (a, bta, k) in enumerate(((0.05, 0.02, 10), (0.1, 0.005, 7), (0.002, 0.3, 12))):
        wi, wd, _ = oidx.knn_query_batch(base, qs, a, bta, k)
        for r in (0, 1):
            ids, dd = res[r][i]
            assert np.array_equal(ids.astype(np.uint32), wi), (r, a, bta, k)
            assert np.array_equal(dd, wd), (r, a, bta, k)


@pytest.mark.gpu
# blocks that are multiples of 2048 (and None = suco_gpu_shard_block_hint) take the
# fused path: select slabs == blocks, histograms written by the select kernel
@pytest.mark.parametrize("G,block", [(1, 4096), (2, 512), (3, 1000), (4, 256), (8, 2048), (1, None), (2, None),
                                     (3, None), (3, 6144)])
def test_gpu_emulated_shards_match_unsharded(gpu, oracle, G, block):
    from paper_2411_14754_b200.sharded import GpuShard, emulate
    full = oracle.clustered(20000 + 50, 32, 40, 77 + G, 20, 140, 18, True)
    base, qs = oracle.hold_out(full, 50, 78)
    idx = gpu.build_index(base, gpu.IndexParams(4, 16, 3, 42))
    shards = [GpuShard(idx, r, G, block) for r in range(G)]
    q = torch.from_numpy(qs).cuda()
    # last case: fewer than m points collide at all, so T = 0 and zero-score ties fill the quota
    for a, b, k in ((0.05, 0.005, 10), (0.02, 0.05, 40), (0.3, 0.001, 3), (0.001, 0.4, 5)):
        want_i, want_d = idx.knn_query_batch(qs, gpu.CollisionParams(a, b, k))
        ids, dd = emulate(shards, q, gpu.CollisionParams(a, b, k))
        assert np.array_equal(ids.cpu().numpy().astype(np.uint32), want_i), (G, block, a, b, k)
        assert np.array_equal(dd.cpu().numpy(), want_d), (G, block, a, b, k)


@pytest.mark.gpu
@pytest.mark.parametrize("G,block", [(1, 4096), (2, 2048), (3, 6144), (4, None), (8, 2048)])
def test_gpu_emulated_split_traversal_matches_unsharded(gpu, oracle, G, block):
    """Query-split protocol: each emulated shard traverses its slice of the batch; phases 1 and 2
    run on the concatenated cell lists (dense select)."""
    from paper_2411_14754_b200.sharded import GpuShard, emulate
    full = oracle.clustered(20000 + 50, 32, 40, 177 + G, 20, 140, 18, True)
    base, qs = oracle.hold_out(full, 50, 178)
    idx = gpu.build_index(base, gpu.IndexParams(4, 16, 3, 42))
    shards = [GpuShard(idx, r, G, block) for r in range(G)]
    assert all(s.split_traversal for s in shards)
    q = torch.from_numpy(qs).cuda()
    for a, b, k in ((0.05, 0.005, 10), (0.02, 0.05, 40), (0.001, 0.4, 5)):
        want_i, want_d = idx.knn_query_batch(qs, gpu.CollisionParams(a, b, k))
        ids, dd = emulate(shards, q, gpu.CollisionParams(a, b, k), split=True)
        assert np.array_equal(ids.cpu().numpy().astype(np.uint32), want_i), (G, block, a, b, k)
        assert np.array_equal(dd.cpu().numpy(), want_d), (G, block, a, b, k)


@pytest.mark.gpu
def test_gpu_shard_float_data(gpu, oracle):
    from paper_2411_14754_b200.sharded import GpuShard, emulate
    base = oracle.clustered(6000, 24, 12, 9, 0.0, 1.0, 0.05, False)
    qs = oracle.uniform(30, 24, 10, 0.0, 1.0)
    idx = gpu.build_index(base, gpu.IndexParams(3, 10, 3, 1, gpu.SubspaceMode.Shuffled))
    shards = [GpuShard(idx, r, 4, 300) for r in range(4)]
    cp = gpu.CollisionParams(0.05, 0.01, 10)
    want_i, want_d = idx.knn_query_batch(qs, cp)
    ids, dd = emulate(shards, torch.from_numpy(qs).cuda(), cp)
    assert np.array_equal(ids.cpu().numpy().astype(np.uint32), want_i)
    assert np.array_equal(dd.cpu().numpy(), want_d)
