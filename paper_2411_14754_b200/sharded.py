"""Multi-GPU SuCo: the block-cyclic shard protocol of libsuco_b200.

The reference is single-host (no distributed API); the library's shard entry
points (include/suco_b200.h, "multi-GPU shard protocol") are the sharded form
of build_index / knn_query and give bit-identical results for any number of
shards. This module is the thin Python mirror of that C-ABI:

  * `Comm` — the communicator: NCCL (`Comm.nccl`, one process per GPU; the
    128-byte NCCL id travels over any out-of-band channel, e.g.
    torch.distributed's broadcast_object_list) or in-process (`Comm.local`,
    G members driven by G host threads — G shards on one GPU for CI);
  * `Shard` — one shard's device index: cut from a full index
    (`Shard.cut`), or built across the ranks from each rank's own rows
    (`Shard.build`: the 2*N_s k-means jobs spread over the ranks);
  * `Shard.knn_query_batch` — every rank passes the same queries and gets the
    full result; inside the library: three all-gathers (per-shard score totals
    -> the global threshold, per-block tie counts -> id-ordered quotas, local
    top-k -> a G-way merge), all on the device, no host round trip.

`run_ranks(fn, G)` drives G in-process ranks on threads (ctypes releases the
GIL inside library calls, so the ranks' collectives meet).
"""
from __future__ import annotations

import ctypes as C
import threading
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

from . import _capi as _c
from . import CollisionParams, GpuIndex, IndexParams, QueryContext, _check, _f32, _p


# ----------------------------------------------------------------- communicators
class Comm:
    """A suco_comm member (one rank)."""

    def __init__(self, handle: C.c_void_p, keep=None):
        self._h = handle
        self._keep = keep

    @classmethod
    def local(cls, nranks: int) -> List["Comm"]:
        """nranks members of one in-process communicator (suco_comm_local_create)."""
        arr = (C.c_void_p * nranks)()
        _check(_c.comm_local_create(nranks, arr))
        return [cls(C.c_void_p(arr[r])) for r in range(nranks)]

    @staticmethod
    def nccl_id() -> bytes:
        buf = np.zeros(128, np.uint8)
        _check(_c.comm_nccl_id(_p(buf, _c.u8p)))
        return buf.tobytes()

    @classmethod
    def nccl(cls, rank: int, size: int, device: int, nccl_id: bytes) -> "Comm":
        """This rank's member of an NCCL communicator (every rank passes rank 0's nccl_id())."""
        buf = np.frombuffer(nccl_id, np.uint8).copy()
        h = C.c_void_p()
        _check(_c.comm_nccl_create(_p(buf, _c.u8p), size, rank, device, C.byref(h)))
        return cls(h)

    @classmethod
    def from_torch(cls, device: int) -> "Comm":
        """NCCL communicator over the ranks of the default torch.distributed group (the id is
        broadcast with broadcast_object_list)."""
        import torch.distributed as dist
        rank, size = dist.get_rank(), dist.get_world_size()
        obj = [cls.nccl_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return cls.nccl(rank, size, device, obj[0])

    @property
    def handle(self):
        return self._h

    def info(self) -> Tuple[int, int, int]:
        r, s, b = C.c_int(), C.c_int(), C.c_uint64()
        _check(_c.comm_info(self._h, C.byref(r), C.byref(s), C.byref(b)))
        return r.value, s.value, b.value

    @property
    def rank(self) -> int:
        return self.info()[0]

    @property
    def size(self) -> int:
        return self.info()[1]

    @property
    def bytes_sent(self) -> int:
        return self.info()[2]

    def close(self):
        if getattr(self, "_h", None):
            _c.comm_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_ranks(fn: Callable[[int], object], nranks: int) -> list:
    """fn(rank) on nranks threads (in-process ranks); returns the results in rank order and
    re-raises the first failure."""
    out: list = [None] * nranks
    err: list = [None] * nranks

    def body(r):
        try:
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001 - re-raised below
            err[r] = e

    ts = [threading.Thread(target=body, args=(r,)) for r in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in err:
        if e is not None:
            raise e
    return out


# ----------------------------------------------------------------- layout
def block_hint(n: int, num_shards: int) -> int:
    """suco_gpu_shard_block_hint: a power of two in [2048, 65536], about n / (100 G)."""
    b = C.c_uint32()
    _check(_c.shard_block_hint(n, num_shards, C.byref(b)))
    return b.value


def shard_ids(n: int, block: int, num_shards: int, shard: int) -> np.ndarray:
    """Global ids of shard `shard`'s rows in its local order (blocks j = shard mod G, id order)."""
    nb = -(-n // block)
    parts = [np.arange(j * block, min(n, (j + 1) * block), dtype=np.int64) for j in range(shard, nb, num_shards)]
    return np.concatenate(parts) if parts else np.zeros(0, np.int64)


# ----------------------------------------------------------------- shards
class Shard(GpuIndex):
    """One block-cyclic shard's device index (layout, all centroids, GLOBAL cell sizes, its own
    rows and local IMI)."""

    @classmethod
    def cut(cls, full: GpuIndex, shard: int, num_shards: int, block: Optional[int] = None) -> "Shard":
        """suco_gpu_make_shard: shard `shard` of num_shards from a full index on the same device."""
        if block is None:
            block = block_hint(full.n, num_shards)
        h = C.c_void_p()
        _check(_c.make_shard(full.handle, shard, num_shards, block, C.byref(h)))
        return cls(h)

    @classmethod
    def build(cls, rows, n_global: int, params: IndexParams, block: int, comm: Comm, device: int = 0,
              train_ids=None) -> "Shard":
        """suco_gpu_build_shard: every rank passes ITS rows (shard_ids(n_global, block, G, rank) of
        the dataset, in that order; a host matrix or a CUDA tensor); k-means jobs run one per rank
        (job j on rank j % G)."""
        if getattr(rows, "is_cuda", False):  # a CUDA float32 tensor: rows stay on the device
            if rows.dtype != __import__("torch").float32 or rows.dim() != 2 or not rows.is_contiguous():
                raise ValueError("device rows must be a contiguous n_local x d float32 tensor")
            ptr, d, r = C.c_void_p(rows.data_ptr()), rows.shape[1], rows
        else:
            r = _f32(rows)
            if r.ndim != 2:
                raise ValueError("rows must be an n_local x d matrix")
            ptr, d = r.ctypes.data_as(C.c_void_p), r.shape[1]
        tr = None if train_ids is None else np.ascontiguousarray(train_ids, np.uint32)
        pc = params._c()
        h = C.c_void_p()
        _check(_c.build_shard(ptr, n_global, d, C.byref(pc), block,
                              _p(tr, _c.u32p) if tr is not None else None, 0 if tr is None else tr.size,
                              comm.handle, device, C.byref(h)))
        return cls(h)

    def shard_info(self):
        ng, nl, b, s, G = C.c_uint64(), C.c_uint64(), C.c_uint32(), C.c_uint32(), C.c_uint32()
        _check(_c.shard_info(self._h, C.byref(ng), C.byref(nl), C.byref(b), C.byref(s), C.byref(G)))
        return {"n_global": ng.value, "n_local": nl.value, "block": b.value, "shard": s.value, "num_shards": G.value}

    def knn_query_batch(self, comm: Comm, queries, params: CollisionParams,  # type: ignore[override]
                        scratch: Optional[QueryContext] = None) -> Tuple[np.ndarray, np.ndarray]:
        """All ranks call this with the same queries; each gets the full (ids nq x k, dists nq x k)."""
        q = _f32(queries)
        if q.ndim == 1:
            q = q[None, :]
        nq, qlen = q.shape
        k = int(params.k)
        ids = np.zeros((nq, max(k, 1)), np.uint32)
        dists = np.zeros((nq, max(k, 1)), np.float64)
        cp = params._c()
        _check(_c.shard_knn_query_batch(self._h, comm.handle, _p(q, _c.f32p), nq, qlen, C.byref(cp),
                                        _p(ids, _c.u32p), _p(dists, _c.f64p), scratch.handle if scratch else None))
        return ids[:, :k], dists[:, :k]

    def knn_query_batch_device(self, comm: Comm, d_queries: int, nq: int, qlen: int,  # type: ignore[override]
                               params: CollisionParams, d_ids: int, d_dists: int, stream: Optional[int] = None,
                               scratch: Optional[QueryContext] = None) -> None:
        cp = params._c()
        _check(_c.shard_knn_query_batch_device(self._h, comm.handle, C.c_void_p(d_queries), nq, qlen, C.byref(cp),
                                               C.c_void_p(d_ids), C.c_void_p(d_dists), C.c_void_p(stream or 0),
                                               scratch.handle if scratch else None))


def emulate(shards: Sequence[Shard], queries, params: CollisionParams):
    """The protocol for G shards in one process (G threads over an in-process communicator):
    every rank's (ids, dists) — all equal by construction."""
    comms = Comm.local(len(shards))
    try:
        return run_ranks(lambda r: shards[r].knn_query_batch(comms[r], queries, params), len(shards))
    finally:
        for c in comms:
            c.close()
