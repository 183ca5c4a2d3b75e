"""Multi-GPU SuCo queries: the block-cyclic shard protocol.

The reference is single-host (no distributed API); this module is the sharded
form of `knn_query` and gives bit-identical results for any number of shards.
Global id block j = [j*b, (j+1)*b) lives on shard j % G. Each shard runs the
C-ABI shard entry points (include/suco_b200.h: suco_gpu_shard_histograms /
suco_gpu_shard_topk) on its own GPU; between them this module does the
exchange — the only cross-shard data the reference's selection needs:

  * per query, the sum over shards of #points with score >= t gives the global
    threshold T = max{t : #(score >= t) >= m} and need = m - #(score > T)
    (query.cpp:242-260: top-m by (score desc, id asc));
  * the per-block tie counts at T, laid out in GLOBAL block order, give each
    block's quota = the first `need` ties in id order (an allreduce of totals
    alone would lose which shard holds the lowest-id ties);
  * every shard re-ranks only its own candidates and returns its top-min(k, c)
    as (squared distance, id); the k smallest pairs over all shards, then sqrt,
    are exactly the reference's result (query.cpp:181-192).

Collectives go through `Comm`: `TorchComm` wraps torch.distributed (NCCL on
GPUs, gloo on CPU for tests); `emulate()` runs G shards in one process (CI on
one GPU, as SURVEY §8(e) suggests). The math is plain torch tensor ops on the
shards' device (small: nq x blocks x (N_s + 2) counters).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import torch

from . import _capi as _c
from . import CollisionParams, GpuIndex, _check, candidate_count


# ----------------------------------------------------------------- exchange math
@dataclass
class Plan:
    T: torch.Tensor       # [nq] u32 threshold score
    quota: torch.Tensor   # [nq, nb_local] ties to take per local block
    base: torch.Tensor    # [nq, nb_local] output offset of each local block
    counts: torch.Tensor  # [nq] local candidates per query
    stride: int           # candidate row length (>= max counts)


def global_threshold(total_ge: torch.Tensor, m: int) -> Tuple[torch.Tensor, torch.Tensor]:
    """total_ge [nq, ns+2] (#score >= t summed over all points) -> (T [nq], need [nq])."""
    ns = total_ge.shape[1] - 2
    t = torch.arange(ns + 2, device=total_ge.device)
    ok = (total_ge >= m) & (t >= 1) & (t <= ns)
    T = torch.where(ok, t.expand_as(ok), torch.zeros_like(t).expand_as(ok)).max(dim=1).values
    gt_total = total_ge.gather(1, (T + 1).unsqueeze(1)).squeeze(1)
    return T, m - gt_total


def piece_order(np_local: int, G: int, r: int, ppb: int, device) -> torch.Tensor:
    """Global position of each of shard r's pieces: local piece p is sub-piece p % ppb of local
    block p // ppb, i.e. of global block (p // ppb) * G + r."""
    p = torch.arange(np_local, device=device)
    return ((p // ppb) * G + r) * ppb + p % ppb


def plan_for_shard(hists: Sequence[torch.Tensor], shard: int, m: int, ppb: int = 1) -> Plan:
    """hists[r] = shard r's [nq, pieces_r, ns+2] piece histograms (all shards' copies); ppb =
    pieces per block (1: the pieces are the blocks)."""
    G = len(hists)
    nq = hists[0].shape[0]
    h64 = [h.to(torch.int64) for h in hists]
    total_ge = sum(h.sum(dim=1) for h in h64)  # [nq, ns+2]
    T, need = global_threshold(total_ge, m)
    Tidx = T.view(nq, 1, 1)
    ties, gts = [], []
    for h in h64:
        at_T = h.gather(2, Tidx.expand(nq, h.shape[1], 1)).squeeze(2)
        above = h.gather(2, (Tidx + 1).expand(nq, h.shape[1], 1)).squeeze(2)
        ties.append(at_T - above)
        gts.append(above)
    # pieces laid out in global id order
    orders = [piece_order(t.shape[1], G, r, ppb, T.device) for r, t in enumerate(ties)]
    width = int(max(int(o.max()) + 1 if o.numel() else 0 for o in orders))
    glob = torch.zeros((nq, max(width, 1)), dtype=torch.int64, device=T.device)
    for o, t in zip(orders, ties):
        glob[:, o] = t
    before = torch.cumsum(glob, dim=1) - glob
    quota_glob = torch.clamp(torch.minimum(glob, need.unsqueeze(1) - before), min=0)
    quota = quota_glob[:, orders[shard]]
    take = gts[shard] + quota
    base = torch.cumsum(take, dim=1) - take
    counts = take.sum(dim=1)
    stride = int(counts.max().item()) if nq else 0
    u32 = torch.int32  # device buffers are read as u32 by the kernels (all values < 2^31)
    return Plan(T.to(u32).contiguous(), quota.to(u32).contiguous(), base.to(u32).contiguous(),
                counts.to(u32).contiguous(), max(stride, 1))


def merge_topk(ids: Sequence[torch.Tensor], sq: Sequence[torch.Tensor], k: int) -> Tuple[torch.Tensor, torch.Tensor]:
    """Per query, the k smallest (squared distance, id) over all shards' lists; sqrt last."""
    I = torch.cat([i.to(torch.int64) & 0xFFFFFFFF for i in ids], dim=1)
    D = torch.cat(list(sq), dim=1)
    o = torch.sort(I, dim=1, stable=True).indices          # secondary key: id
    I, D = I.gather(1, o), D.gather(1, o)
    o = torch.sort(D, dim=1, stable=True).indices          # primary key: squared distance
    I, D = I.gather(1, o)[:, :k], D.gather(1, o)[:, :k]
    return I.to(torch.int64), ieee_sqrt(D)


def ieee_sqrt(D: torch.Tensor) -> torch.Tensor:
    """Correctly rounded sqrt (std::sqrt / query.cpp:192). CUDA's double sqrt is IEEE;
    torch's CPU float64 sqrt is not (vectorised, ~1 ulp), so CPU tensors go through numpy."""
    if D.is_cuda:
        return torch.sqrt(D)
    import numpy as np
    return torch.from_numpy(np.sqrt(D.numpy()))


# ----------------------------------------------------------------- GPU shard
def _torch_stream(device) -> int:
    """torch's current stream as a cudaStream_t for the C-ABI. Handle 0 (the legacy
    default stream) would mean "the index's own stream" there, so it maps to
    cudaStreamLegacy (1)."""
    return torch.cuda.current_stream(device).cuda_stream or 1


def block_hint(full: GpuIndex, num_shards: int) -> int:
    """Fastest block size for `num_shards` shards (suco_gpu_shard_block_hint): slabs == blocks."""
    b = C.c_uint32()
    _check(_c.shard_block_hint(full.handle, num_shards, C.byref(b)))
    return b.value


class GpuShard:
    """One block-cyclic shard of a device index (suco_gpu_make_shard); block=None picks block_hint."""

    def __init__(self, full: GpuIndex, shard: int, num_shards: int, block: Optional[int] = None):
        if block is None:
            block = block_hint(full, num_shards)
        h = C.c_void_p()
        _check(_c.make_shard(full.handle, shard, num_shards, block, C.byref(h)))
        self.index = GpuIndex(h)
        ng, nl, nb, b, s, G = (C.c_uint64(), C.c_uint64(), C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_uint32())
        _check(_c.shard_info(h, C.byref(ng), C.byref(nl), C.byref(nb), C.byref(b), C.byref(s), C.byref(G)))
        self.n_global, self.n_local, self.nblocks = ng.value, nl.value, nb.value
        self.block, self.shard, self.num_shards = b.value, s.value, G.value
        self.ns = full.params.num_subspaces
        self.d = full.d
        ppb, dense = C.c_uint32(), C.c_int()
        _check(_c.shard_pieces(h, C.byref(ppb), C.byref(dense)))
        self.ppb = ppb.value  # histogram pieces per block (dense select: 2048-id pieces)
        self.dense = bool(dense.value)
        self.K = full.params.k_half ** 2

    def histograms(self, q: torch.Tensor, params: CollisionParams, stream: Optional[int] = None) -> torch.Tensor:
        stream = stream or _torch_stream(q.device)  # ordered with the plan math
        nq = q.shape[0]
        hist = torch.empty((nq, self.nblocks, self.ns + 2), dtype=torch.int32, device=q.device)
        cp = params._c()
        _check(_c.shard_histograms(self.index.handle, C.c_void_p(q.data_ptr()), nq, self.d, C.byref(cp),
                                   C.c_void_p(hist.data_ptr()), C.c_void_p(stream or 0)))
        return hist

    def topk(self, q: torch.Tensor, params: CollisionParams, plan: Plan, stream: Optional[int] = None):
        stream = stream or _torch_stream(q.device)
        nq, k = q.shape[0], int(params.k)
        ids = torch.empty((nq, k), dtype=torch.int32, device=q.device)
        sq = torch.empty((nq, k), dtype=torch.float64, device=q.device)
        cp = params._c()
        _check(_c.shard_topk(self.index.handle, C.c_void_p(q.data_ptr()), nq, self.d, C.byref(cp),
                             C.c_void_p(plan.T.data_ptr()), C.c_void_p(plan.quota.data_ptr()),
                             C.c_void_p(plan.base.data_ptr()), C.c_void_p(plan.counts.data_ptr()), plan.stride,
                             C.c_void_p(ids.data_ptr()), C.c_void_p(sq.data_ptr()), C.c_void_p(stream or 0)))
        return ids, sq


    # ---- query-split traversal (multi-GPU): every rank traverses a slice of the batch
    @property
    def split_traversal(self) -> bool:
        """The query-split protocol needs the dense select (its phases take exchanged cell lists)."""
        return self.dense

    def traverse_slice(self, q: torch.Tensor, params: CollisionParams, stream: Optional[int] = None):
        """Traversal of this rank's query slice -> (compact cells u32 [L], counts [nq_slice, ns])."""
        stream = stream or _torch_stream(q.device)
        nq = q.shape[0]
        K = self.K
        cells = torch.empty((max(nq, 1), self.ns, K), dtype=torch.int32, device=q.device)
        ncells = torch.zeros((max(nq, 1), self.ns), dtype=torch.int32, device=q.device)
        if nq:
            cp = params._c()
            _check(_c.shard_traverse(self.index.handle, C.c_void_p(q.data_ptr()), nq, self.d, C.byref(cp),
                                     C.c_void_p(cells.data_ptr()), C.c_void_p(ncells.data_ptr()), C.c_void_p(stream)))
        cells, ncells = cells[:nq], ncells[:nq]
        keep = torch.arange(K, device=q.device).view(1, 1, K) < ncells.unsqueeze(2)
        return cells[keep], ncells

    def histograms_cells(self, nq: int, params: CollisionParams, cells: torch.Tensor, off: torch.Tensor,
                         stream: Optional[int] = None) -> torch.Tensor:
        stream = stream or _torch_stream(cells.device)
        hist = torch.empty((nq, self.nblocks, self.ns + 2), dtype=torch.int32, device=cells.device)
        cp = params._c()
        _check(_c.shard_histograms_cells(self.index.handle, nq, C.byref(cp), C.c_void_p(cells.data_ptr()),
                                         C.c_void_p(off.data_ptr()), C.c_void_p(hist.data_ptr()), C.c_void_p(stream)))
        return hist

    def topk_cells(self, q: torch.Tensor, params: CollisionParams, plan: Plan, cells: torch.Tensor,
                   off: torch.Tensor, stream: Optional[int] = None):
        stream = stream or _torch_stream(q.device)
        nq, k = q.shape[0], int(params.k)
        ids = torch.empty((nq, k), dtype=torch.int32, device=q.device)
        sq = torch.empty((nq, k), dtype=torch.float64, device=q.device)
        cp = params._c()
        _check(_c.shard_topk_cells(self.index.handle, C.c_void_p(q.data_ptr()), nq, self.d, C.byref(cp),
                                   C.c_void_p(cells.data_ptr()), C.c_void_p(off.data_ptr()),
                                   C.c_void_p(plan.T.data_ptr()), C.c_void_p(plan.quota.data_ptr()),
                                   C.c_void_p(plan.base.data_ptr()), C.c_void_p(plan.counts.data_ptr()), plan.stride,
                                   C.c_void_p(ids.data_ptr()), C.c_void_p(sq.data_ptr()), C.c_void_p(stream)))
        return ids, sq


def query_slice(nq: int, rank: int, size: int) -> Tuple[int, int]:
    """Rank `rank`'s contiguous slice of a batch of nq queries."""
    return nq * rank // size, nq * (rank + 1) // size


def cell_offsets(ncells: torch.Tensor) -> torch.Tensor:
    """[nq, ns] counts -> nq*ns + 1 u64 offsets into the compact cell array."""
    off = torch.zeros(ncells.numel() + 1, dtype=torch.int64, device=ncells.device)
    off[1:] = torch.cumsum(ncells.reshape(-1).to(torch.int64), dim=0)
    return off


# ----------------------------------------------------------------- protocols
class TorchComm:
    """torch.distributed collectives (NCCL for CUDA tensors, gloo for CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def allgather_var(self, t: torch.Tensor) -> List[torch.Tensor]:
        """all_gather of tensors whose dim 1 may differ per rank (padded on the wire)."""
        d1 = torch.tensor([t.shape[1]], dtype=torch.int64, device=t.device)
        sizes = [torch.zeros_like(d1) for _ in range(self.size)]
        self.dist.all_gather(sizes, d1, group=self.group)
        mx = int(max(s.item() for s in sizes))
        pad = torch.zeros((t.shape[0], mx) + tuple(t.shape[2:]), dtype=t.dtype, device=t.device)
        pad[:, : t.shape[1]] = t
        out = [torch.empty_like(pad) for _ in range(self.size)]
        self.dist.all_gather(out, pad.contiguous(), group=self.group)
        return [o[:, : int(s.item())] for o, s in zip(out, sizes)]


def knn_query_distributed(engine, comm: TorchComm, queries: torch.Tensor, params: CollisionParams):
    """Every rank calls this with the same queries; returns the global (ids int64 [nq,k], dists f64 [nq,k]).
    Engines with `split_traversal` traverse only their slice of the batch and exchange the cell lists."""
    m = candidate_count(params.beta, engine.n_global, params.k)
    if getattr(engine, "split_traversal", False):
        nq = queries.shape[0]
        lo, hi = query_slice(nq, comm.rank, comm.size)
        mine, nc = engine.traverse_slice(queries[lo:hi], params)
        cells = torch.cat(comm.allgather_var(mine.view(1, -1)), dim=1).view(-1)
        ncells = torch.cat([t.t() for t in comm.allgather_var(nc.t().contiguous())], dim=0)
        off = cell_offsets(ncells)
        hist = engine.histograms_cells(nq, params, cells, off)
        hists = comm.allgather_var(hist)
        plan = plan_for_shard(hists, comm.rank, m, getattr(engine, "ppb", 1))
        ids, sq = engine.topk_cells(queries, params, plan, cells, off)
        all_ids = comm.allgather_var(ids)
        all_sq = comm.allgather_var(sq)
        return merge_topk(all_ids, all_sq, int(params.k))
    hist = engine.histograms(queries, params)
    hists = comm.allgather_var(hist)
    plan = plan_for_shard(hists, comm.rank, m, getattr(engine, "ppb", 1))
    ids, sq = engine.topk(queries, params, plan)
    all_ids = comm.allgather_var(ids)
    all_sq = comm.allgather_var(sq)
    return merge_topk(all_ids, all_sq, int(params.k))


def emulate(engines: Sequence, queries: torch.Tensor, params: CollisionParams, split: bool = False):
    """Run the protocol for G shard engines in one process (single-GPU CI of the multi-GPU path);
    split=True: each engine traverses its slice of the batch and the cell lists are concatenated."""
    m = candidate_count(params.beta, engines[0].n_global, params.k)
    if split:
        G, nq = len(engines), queries.shape[0]
        parts = [e.traverse_slice(queries[slice(*query_slice(nq, r, G))], params) for r, e in enumerate(engines)]
        cells = torch.cat([p[0] for p in parts])
        off = cell_offsets(torch.cat([p[1] for p in parts]))
        hists = [e.histograms_cells(nq, params, cells, off) for e in engines]
        tops = [e.topk_cells(queries, params, plan_for_shard(hists, r, m, e.ppb), cells, off)
                for r, e in enumerate(engines)]
        return merge_topk([t[0] for t in tops], [t[1] for t in tops], int(params.k))
    hists = [e.histograms(queries, params) for e in engines]
    tops = [e.topk(queries, params, plan_for_shard(hists, r, m, getattr(e, "ppb", 1))) for r, e in enumerate(engines)]
    return merge_topk([t[0] for t in tops], [t[1] for t in tops], int(params.k))
