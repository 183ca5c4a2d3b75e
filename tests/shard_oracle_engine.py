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


class OracleSplitShard(OracleShard):
    """OracleShard with the query-split traversal interface. The C oracle does not expose its
    retrieved-cell lists, so traverse_slice returns a stand-in payload per (query, subspace):
    as many entries as the oracle retrieves, with values derived from the query. histograms_cells
    asserts that the payload gathered from every rank is exactly each query's own (the exchange
    and offset plumbing), then scores the shard with the oracle."""

    split_traversal = True

    def _payload(self, qrow, cps):
        tag = int(np.abs(qrow).sum() * 1000) % 1000003
        return [np.arange(c, dtype=np.int64) * 7 + tag * 31 + s for s, c in enumerate(cps)]

    def _cps(self, qrow, params):
        _, _, cps, _ = self.idx.query_intermediates(self.data, qrow, params.alpha, params.beta, params.k)
        return cps

    def traverse_slice(self, q, params):
        qs = q.numpy()
        parts, counts = [], np.zeros((len(qs), self.ns), np.int32)
        for i, row in enumerate(qs):
            cps = self._cps(row, params)
            counts[i] = cps
            parts.extend(self._payload(row, cps))
        flat = np.concatenate(parts) if parts else np.zeros(0, np.int64)
        return torch.from_numpy(flat.astype(np.int32)), torch.from_numpy(counts)

    def _check_cells(self, queries, params, cells, off):
        cells, off = cells.numpy(), off.numpy()
        for i, row in enumerate(queries.numpy()):
            want = self._payload(row, self._cps(row, params))
            for s in range(self.ns):
                got = cells[off[i * self.ns + s]: off[i * self.ns + s + 1]]
                assert np.array_equal(got, want[s].astype(np.int32)), (i, s)

    def histograms_cells(self, nq, params, cells, off):
        self._check_cells(self._queries, params, cells, off)
        return self.histograms(self._queries, params)

    def topk_cells(self, q, params, plan, cells, off):
        self._check_cells(q, params, cells, off)
        return self.topk(q, params, plan)
