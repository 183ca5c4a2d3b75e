"""TEST INFRASTRUCTURE: a CPU shard engine backed by the C oracle.

Implements the same two-phase contract as paper_2411_14754_b200.sharded.GpuShard
(histograms -> plan -> topk) for one block-cyclic shard, so the exchange math and
the torch.distributed plumbing can be tested with gloo on CPU (world_size 2) and
compared bit-for-bit with the unsharded oracle.
"""
import numpy as np
import torch


class OracleShard:
    def __init__(self, oracle, oidx, data, shard, num_shards, block):
        self.O, self.idx, self.data = oracle, oidx, np.ascontiguousarray(data, np.float32)
        self.n_global, self.d = self.data.shape
        self.shard, self.num_shards, self.block = shard, num_shards, block
        nb = -(-self.n_global // block)
        self.blocks = [j for j in range(nb) if j % num_shards == shard]
        self.local_ids = np.concatenate([np.arange(j * block, min(self.n_global, (j + 1) * block)) for j in self.blocks])
        self.n_local = self.local_ids.size
        self.nblocks = len(self.blocks)
        self.ns = oidx.info()[2]
        self._scores = None

    def histograms(self, q: torch.Tensor, params) -> torch.Tensor:
        qs = q.numpy()
        hist = np.zeros((len(qs), self.nblocks, self.ns + 2), np.int32)
        self._scores = []
        for i, row in enumerate(qs):
            scores, _, _, _ = self.idx.query_intermediates(self.data, row, params.alpha, params.beta, params.k)
            self._scores.append(scores)
            for bi, j in enumerate(self.blocks):
                s = scores[j * self.block: min(self.n_global, (j + 1) * self.block)]
                for t in range(self.ns + 2):
                    hist[i, bi, t] = int((s >= t).sum()) if t <= self.ns else 0
        return torch.from_numpy(hist)

    def topk(self, q: torch.Tensor, params, plan):
        qs = q.numpy()
        k = int(params.k)
        ids = np.full((len(qs), k), 0xFFFFFFFF, np.uint32)
        sq = np.full((len(qs), k), np.inf, np.float64)
        T = plan.T.numpy()
        quota = plan.quota.numpy()
        for i, row in enumerate(qs):
            scores = self._scores[i]
            cands = []
            for bi, j in enumerate(self.blocks):
                lo, hi = j * self.block, min(self.n_global, (j + 1) * self.block)
                s = scores[lo:hi]
                gt = np.nonzero(s > T[i])[0] + lo
                ties = (np.nonzero(s == T[i])[0] + lo)[: int(quota[i, bi])]
                cands.extend(gt.tolist() + ties.tolist())
            assert len(cands) == int(plan.counts[i])
            pairs = sorted((self.O.sqdist4(self.data[c], row), c) for c in cands)[:k]
            for r, (dd, c) in enumerate(pairs):
                ids[i, r], sq[i, r] = c, dd
        return torch.from_numpy(ids.view(np.int32)), torch.from_numpy(sq)
