"""TEST INFRASTRUCTURE: a CPU model of the library's multi-GPU shard protocol.

A statement-for-statement Python restatement of what one rank of
libsuco_b200's sharded query does (capi_shard.cu shard_run + the dense.cu
shard kernels shard_totals / shard_ties / shard_quota, shard.cu merge_topk),
with the SC-scores and exact distances supplied by the C oracle. It runs over
any all-gather: torch.distributed (gloo, world_size 2, on CPU) or an
in-process stand-in, so the exchange rounds and their id-ordered tie rule are
checked on the CPU against the unsharded reference results. The GPU tests
check the library itself against the oracle.

Per query batch:
  1. per-shard totals #(score >= t), t = 1..16          -> all-gather
  2. T = max{t <= N_s : sum >= m}, need = m - #(score > T);
     per local block: ties at T                         -> all-gather
  3. quota of global block j (shard j % G, local j // G) = the first `need`
     ties in global id order; per local piece: its share in id order;
     candidates = score > T plus the quota ties
  4. local top-k by (squared distance, id)              -> all-gather
  5. k smallest (squared distance, id) over the shards, sqrt.
"""
from __future__ import annotations

import numpy as np

LEVELS = 16


class ModelShard:
    """Shard r of G over n points: blocks of `block` ids, pieces of `piece` ids (block % piece == 0)."""

    def __init__(self, oracle, oidx, data, shard, num_shards, block, piece):
        assert block % piece == 0
        self.O, self.idx, self.data = oracle, oidx, np.ascontiguousarray(data, np.float32)
        self.n, self.d = self.data.shape
        self.r, self.G, self.b, self.wp = shard, num_shards, block, piece
        self.nb = -(-self.n // block)
        self.blocks = list(range(shard, self.nb, num_shards))
        self.nbl_max = -(-self.nb // num_shards)
        self.ns = oidx.info()[2]
        # local pieces (global lo, hi) in local order, and each piece's local block
        self.pieces, self.piece_block = [], []
        for lb, j in enumerate(self.blocks):
            lo = j * block
            while lo < min(self.n, (j + 1) * block):
                self.pieces.append((lo, min(self.n, lo + piece, (j + 1) * block)))
                self.piece_block.append(lb)
                lo += piece

    def scores(self, q, params):
        """SC-scores of every point (the shard reads only its own pieces)."""
        s, _, _, _ = self.idx.query_intermediates(self.data, q, params.alpha, params.beta, params.k)
        return s

    def query(self, queries, params, m, allgather):
        """allgather(np.ndarray) -> list of every rank's array (rank order)."""
        nq, k = len(queries), int(params.k)
        sc = [self.scores(q, params) for q in queries]
        # 1. totals
        tot = np.zeros((nq, LEVELS), np.int64)
        for i in range(nq):
            for lo, hi in self.pieces:
                s = sc[i][lo:hi]
                for t in range(1, LEVELS + 1):
                    tot[i, t - 1] += int((s >= t).sum())
        ge = sum(allgather(tot))
        # 2. T, need; ties per local block
        T = np.zeros(nq, np.int64)
        need = np.zeros(nq, np.int64)
        ties = np.zeros((nq, self.nbl_max), np.int64)
        for i in range(nq):
            for t in range(min(self.ns, LEVELS), 0, -1):
                if ge[i, t - 1] >= m:
                    T[i] = t
                    break
            gt_total = ge[i, T[i]] if T[i] + 1 <= self.ns else 0
            need[i] = m - gt_total
            for (lo, hi), lb in zip(self.pieces, self.piece_block):
                ties[i, lb] += int((sc[i][lo:hi] == T[i]).sum())
        ties_all = allgather(ties)
        # 3. quotas in global id order, candidates
        out_ids = np.full((nq, k), 0xFFFFFFFF, np.int64)
        out_sq = np.full((nq, k), np.inf, np.float64)
        for i in range(nq):
            before, qblk = 0, {}
            for j in range(self.nb):
                t = int(ties_all[j % self.G][i, j // self.G])
                quota = 0 if before >= need[i] else min(t, int(need[i] - before))
                if j % self.G == self.r:
                    qblk[j // self.G] = quota
                before += t
            left = dict(qblk)
            cands = []
            for (lo, hi), lb in zip(self.pieces, self.piece_block):
                s = sc[i][lo:hi]
                eq = np.nonzero(s == T[i])[0]
                take = min(len(eq), left[lb])
                left[lb] -= take
                cands += (np.nonzero(s > T[i])[0] + lo).tolist() + (eq[:take] + lo).tolist()
            # 4. local top-k by (squared distance, id)
            pairs = sorted((self.O.sqdist4(self.data[c], queries[i]), c) for c in cands)[:k]
            for r, (dd, c) in enumerate(pairs):
                out_ids[i, r], out_sq[i, r] = c, dd
        all_ids, all_sq = allgather(out_ids), allgather(out_sq)
        # 5. merge
        ids = np.zeros((nq, k), np.uint32)
        dists = np.zeros((nq, k), np.float64)
        for i in range(nq):
            pool = sorted((float(all_sq[g][i, r]), int(all_ids[g][i, r])) for g in range(self.G) for r in range(k))
            for r, (dd, c) in enumerate(pool[:k]):
                ids[i, r], dists[i, r] = c, np.sqrt(dd)
        return ids, dists


def torch_allgather(a: np.ndarray):
    """all_gather over the default torch.distributed group (gloo on CPU)."""
    import torch
    import torch.distributed as dist
    t = torch.from_numpy(np.ascontiguousarray(a))
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [o.numpy() for o in out]


def run_inprocess(shards, queries, params, m):
    """All G model ranks in one process: each all-gather collects every rank's contribution."""
    import threading
    G = len(shards)
    bar = threading.Barrier(G)
    results = [None] * G
    rounds = {}

    def allgather_for(r):
        step = [0]

        def ag(a):
            key = step[0]
            step[0] += 1
            with lock:
                rounds.setdefault(key, [None] * G)[r] = a
            bar.wait()
            got = list(rounds[key])
            bar.wait()
            return got
        return ag

    lock = threading.Lock()

    def body(r):
        results[r] = shards[r].query(queries, params, m, allgather_for(r))

    ts = [threading.Thread(target=body, args=(r,)) for r in range(G)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return results
