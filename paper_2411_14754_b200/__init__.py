"""SuCo on B200: the reference's index-build and batched-query API, on sm_100a kernels.

Python mirror of the reference library's public interface (/root/reference/proj/include/suco):
same names, argument meaning, defaults and error taxonomy, so tests written
against the reference read the same here. Everything below calls the C-ABI of
libsuco_b200.so (include/suco_b200.h); numpy arrays are only host buffers.

    suco.IndexParams        index.hpp:53-61         suco.build_index      index.hpp:85
    suco.CollisionParams    sc_linear.hpp:22-31     suco.knn_query        query.hpp:93-96
    suco.collision_count    sc_linear.hpp:36        suco.rerank           query.hpp:83-84
    suco.candidate_count    sc_linear.hpp:40        suco.centroid_distances query.hpp:27-28
    suco.kmeans             kmeans.hpp:46-48        suco.dynamic_activation query.hpp:57-58
    suco.build_imi          index.hpp:38-39         suco.load_index / GpuIndex.serialize  index.hpp:99-108
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass
from typing import List, NamedTuple, Optional, Tuple

import numpy as np

from . import _capi as _c

__all__ = [
    "Error", "ContractError", "ConfigError", "FormatError", "CorruptIndexError", "IncompatibilityError",
    "SubspaceMode", "IndexParams", "CollisionParams", "Dataset", "Neighbor", "RetrievedCell", "GpuIndex",
    "collision_count", "candidate_count", "build_index", "load_index", "knn_query", "centroid_distances",
    "dynamic_activation", "rerank", "kmeans", "build_imi", "device_count", "QueryContext",
]


# ------------------------------------------------------------------ errors (error.hpp:9-37)
class Error(RuntimeError):
    pass


class ContractError(Error):
    pass


class ConfigError(Error):
    pass


class FormatError(Error):
    pass


class CorruptIndexError(FormatError):
    pass


class IncompatibilityError(Error):
    pass


_CODES = {1: Error, 2: ConfigError, 3: FormatError, 4: IncompatibilityError, 5: ContractError, 6: CorruptIndexError}


def _check(rc: int):
    if rc != 0:
        raise _CODES.get(rc, Error)(_c.last_error().decode(errors="replace"))


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def device_count() -> int:
    n = C.c_int(0)
    _check(_c.device_count(C.byref(n)))
    return n.value


# ------------------------------------------------------------------ params
class SubspaceMode(enum.IntEnum):
    Contiguous = 0
    Shuffled = 1


@dataclass
class IndexParams:
    num_subspaces: int = 8
    k_half: int = 50
    iterations: int = 10
    seed: int = 42
    mode: SubspaceMode = SubspaceMode.Contiguous

    def _c(self) -> _c.IndexParamsC:
        return _c.IndexParamsC(self.num_subspaces, self.k_half, self.iterations, int(self.mode), self.seed)


@dataclass
class CollisionParams:
    alpha: float = 0.05
    beta: float = 0.005
    k: int = 50

    def _c(self) -> _c.CollisionParamsC:
        return _c.CollisionParamsC(float(self.alpha), float(self.beta), int(self.k))

    def validate(self, n: int) -> None:
        """sc_linear.cpp:26-37 — ConfigError unless 0<alpha<=1, 0<beta<=1, 1<=k<=n."""
        cp = self._c()
        _check(_c.validate_collision_params(C.byref(cp), n))


def collision_count(alpha: float, n: int) -> int:
    """max(1, floor(alpha*n)) with 1e-6 snapping (sc_linear.cpp:39-42)."""
    return int(_c.collision_count(alpha, n))


def candidate_count(beta: float, n: int, k: int) -> int:
    """max(k, ceil(beta*n)) with 1e-6 snapping (sc_linear.cpp:44-47)."""
    return int(_c.candidate_count(beta, n, k))


class Dataset:
    """Row-major n x d float32 matrix (core.hpp:17-37); validated on upload."""

    def __init__(self, values):
        v = _f32(values)
        if v.ndim != 2:
            raise ContractError("dataset must be a 2-D n x d matrix")
        self.values = v

    @property
    def n(self) -> int:
        return self.values.shape[0]

    @property
    def d(self) -> int:
        return self.values.shape[1]

    def size(self) -> int:
        return self.n

    def dim(self) -> int:
        return self.d

    def row(self, i: int) -> np.ndarray:
        return self.values[i]


def _values(ds) -> np.ndarray:
    return ds.values if isinstance(ds, Dataset) else _f32(ds)


class Neighbor(NamedTuple):
    id: int
    distance: float


class RetrievedCell(NamedTuple):
    c1: int
    c2: int
    cumulative: int
    sum_dist: float


# ------------------------------------------------------------------ index
class GpuIndex:
    """Device-resident SucoIndex (index.hpp:67-74) plus the dataset rows it re-ranks."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle

    def close(self):
        if getattr(self, "_h", None):
            _c.free_index(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def info(self):
        n = C.c_uint64()
        d = C.c_uint32()
        p = _c.IndexParamsC()
        _check(_c.index_info(self._h, C.byref(n), C.byref(d), C.byref(p), None, None, None))
        return n.value, d.value, IndexParams(p.num_subspaces, p.k_half, p.iterations, p.seed, SubspaceMode(p.mode))

    @property
    def n(self) -> int:
        return self.info()[0]

    @property
    def d(self) -> int:
        return self.info()[1]

    @property
    def params(self) -> IndexParams:
        return self.info()[2]

    def layout(self):
        n, d, p = self.info()
        dims = np.empty(d, np.uint32)
        sizes = np.empty(p.num_subspaces, np.uint32)
        split = np.empty(p.num_subspaces, np.uint32)
        _check(_c.index_info(self._h, None, None, None, _p(dims, _c.u32p), _p(sizes, _c.u32p), _p(split, _c.u32p)))
        return dims, sizes, split

    def subspace(self, s: int):
        """(centroids_first, centroids_second, imi_offsets, imi_ids) of subspace s."""
        n, d, p = self.info()
        _, sizes, split = self.layout()
        h1, h2 = int(split[s]), int(sizes[s] - split[s])
        c1 = np.empty((p.k_half, h1), np.float32)
        c2 = np.empty((p.k_half, h2), np.float32)
        off = np.empty(p.k_half * p.k_half + 1, np.uint64)
        ids = np.empty(n, np.uint32)
        _check(_c.index_subspace(self._h, s, _p(c1, _c.f32p), _p(c2, _c.f32p), _p(off, _c.u64p), _p(ids, _c.u32p)))
        return c1, c2, off, ids

    def serialize(self) -> bytes:
        """serialize_index (index.cpp:147-170): byte-identical to the reference."""
        ln = C.c_uint64()
        _check(_c.serialize_index(self._h, None, 0, C.byref(ln)))
        buf = np.empty(ln.value, np.uint8)
        _check(_c.serialize_index(self._h, _p(buf, _c.u8p), ln.value, C.byref(ln)))
        return buf.tobytes()

    def save(self, path: str) -> None:
        with open(path, "wb") as f:
            f.write(self.serialize())

    def knn_query_batch(self, queries, params: CollisionParams,
                        scratch: Optional["QueryContext"] = None) -> Tuple[np.ndarray, np.ndarray]:
        """Batched knn_query (run_suco_batch, suco_cli.cpp:95-114): (ids nq x k, distances nq x k).
        `scratch`: a QueryContext of this index (the reference's QueryScratch*), or None (pooled)."""
        q = _f32(queries)
        if q.ndim == 1:
            q = q[None, :]
        nq, qlen = q.shape
        k = int(params.k)
        ids = np.zeros((nq, max(k, 1)), np.uint32)
        dists = np.zeros((nq, max(k, 1)), np.float64)
        cp = params._c()
        _check(_c.knn_query_batch(self._h, _p(q, _c.f32p), nq, qlen, C.byref(cp), _p(ids, _c.u32p),
                                  _p(dists, _c.f64p), scratch.handle if scratch else None))
        return ids[:, :k], dists[:, :k]

    def context(self) -> "QueryContext":
        """A new query context (suco_gpu_query_ctx_create) bound to this index."""
        return QueryContext(self)

    def exact_knn_batch(self, queries, k: int) -> Tuple[np.ndarray, np.ndarray]:
        """exact_knn (eval.hpp:29, eval.cpp:28-62) for every row on the GPU: (ids nq x k, distances
        nq x k), ascending by (distance, id) — the ground truth for recall / mre."""
        q = _f32(queries)
        if q.ndim == 1:
            q = q[None, :]
        nq, qlen = q.shape
        ids = np.zeros((nq, max(k, 1)), np.uint32)
        dists = np.zeros((nq, max(k, 1)), np.float64)
        _check(_c.exact_knn_batch(self._h, _p(q, _c.f32p), nq, qlen, int(k), _p(ids, _c.u32p), _p(dists, _c.f64p)))
        return ids[:, :k], dists[:, :k]

    def sc_scores(self, query, alpha: float) -> np.ndarray:
        """compute_sc_scores (sc_linear.cpp:49-93) on the GPU: per point, the number of subspaces in which
        it is among the collision_count(alpha, n) nearest (exact fp64, ties by id). u32 array of n."""
        q = _f32(query).reshape(-1)
        n = self.n
        out = np.zeros(max(n, 1), np.uint32)
        _check(_c.sc_scores(self._h, _p(q, _c.f32p), q.shape[0], float(alpha), _p(out, _c.u32p)))
        return out[:n]

    def sc_linear_batch(self, queries, params: CollisionParams) -> Tuple[np.ndarray, np.ndarray]:
        """sc_linear_query (sc_linear.cpp:95-121) for every row on the GPU — the index-free SC-Linear
        baseline: (ids nq x k, distances nq x k)."""
        q = _f32(queries)
        if q.ndim == 1:
            q = q[None, :]
        nq, qlen = q.shape
        k = int(params.k)
        ids = np.zeros((nq, max(k, 1)), np.uint32)
        dists = np.zeros((nq, max(k, 1)), np.float64)
        cp = params._c()
        _check(_c.sc_linear_batch(self._h, _p(q, _c.f32p), nq, qlen, C.byref(cp), _p(ids, _c.u32p),
                                  _p(dists, _c.f64p)))
        return ids[:, :k], dists[:, :k]

    def knn_query_batch_device(self, d_queries: int, nq: int, qlen: int, params: CollisionParams, d_ids: int,
                               d_dists: int, stream: Optional[int] = None,
                               scratch: Optional["QueryContext"] = None) -> None:
        """Device-resident variant: raw device pointers (e.g. torch tensor .data_ptr()). `stream` is a
        cudaStream_t handle; None / 0 = the context's own stream (pass 1 = cudaStreamLegacy for
        torch's default stream). Returns once enqueued."""
        cp = params._c()
        _check(_c.knn_query_batch_device(self._h, C.c_void_p(d_queries), nq, qlen, C.byref(cp), C.c_void_p(d_ids),
                                         C.c_void_p(d_dists), C.c_void_p(stream or 0),
                                         scratch.handle if scratch else None))

    def query_intermediates(self, query, params: CollisionParams):
        """(scores n, candidates ascending, cells per subspace, cumulative per subspace) of one query."""
        q = _f32(query).ravel()
        n, d, p = self.info()
        scores = np.empty(n, np.uint32)
        cands = np.empty(n, np.uint32)
        m = C.c_uint64()
        cps = np.empty(p.num_subspaces, np.uint32)
        cum = np.empty(p.num_subspaces, np.uint64)
        cp = params._c()
        _check(_c.query_intermediates(self._h, _p(q, _c.f32p), q.size, C.byref(cp), _p(scores, _c.u32p),
                                      _p(cands, _c.u32p), C.byref(m), _p(cps, _c.u32p), _p(cum, _c.u64p)))
        return scores, cands[: m.value].copy(), cps, cum


class QueryContext:
    """Caller-owned query state (suco_gpu_query_ctx; the reference's QueryScratch, query.hpp:72-78):
    pipeline scratch, streams and events, profiling counters. One thread at a time."""

    def __init__(self, index: GpuIndex):
        h = C.c_void_p()
        _check(_c.query_ctx_create(index.handle, C.byref(h)))
        self._h = h
        self.index = index  # keeps the index alive

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            _c.query_ctx_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self) -> None:
        _check(_c.query_ctx_synchronize(self._h))

    def set_profiling(self, enabled: bool) -> None:
        _check(_c.query_ctx_set_profiling(self._h, int(bool(enabled))))

    def stage_times(self):
        """(ms per stage [traverse, select, rerank], retrieved ids summed over queries x subspaces, nq, m)
        of the last query call; needs set_profiling(True) before that call."""
        ms = np.zeros(3, np.float64)
        st = np.zeros(3, np.uint64)
        _check(_c.query_ctx_stage_times(self._h, _p(ms, _c.f64p), _p(st, _c.u64p)))
        return ms, int(st[0]), int(st[1]), int(st[2])

    def last_launches(self) -> int:
        """Kernels (all this library's) the last query call through this context enqueued."""
        n = C.c_uint64()
        _check(_c.query_ctx_last_launches(self._h, C.byref(n)))
        return n.value

    def exchange_bytes(self) -> int:
        """Bytes this rank sent through the communicator in the last shard query."""
        n = C.c_uint64()
        _check(_c.query_ctx_exchange_bytes(self._h, C.byref(n)))
        return n.value


def _rows(dataset):
    """(f32 pointer, n, d, keep-alive) for a host matrix or a CUDA float32 tensor (any object with
    data_ptr() / is_cuda: its rows are copied device to device, never through the host)."""
    if getattr(dataset, "is_cuda", False):
        t = dataset
        if t.dim() != 2 or not t.is_contiguous() or str(t.dtype) != "torch.float32":
            raise ContractError("device dataset must be a contiguous 2-D float32 tensor")
        return C.cast(C.c_void_p(t.data_ptr()), _c.f32p), t.shape[0], t.shape[1], t
    v = _values(dataset)
    if v.ndim != 2:
        raise ContractError("dataset must be a 2-D n x d matrix")
    return _p(v, _c.f32p), v.shape[0], v.shape[1], v


def build_index(dataset, params: IndexParams = IndexParams(), device: int = 0) -> GpuIndex:
    """build_index (index.hpp:85, index.cpp:98-145) on the GPU. `dataset`: host n x d matrix or a
    CUDA float32 tensor on `device`."""
    ptr, n, d, _keep = _rows(dataset)
    h = C.c_void_p()
    ip = params._c()
    _check(_c.build_index(ptr, n, d, C.byref(ip), device, C.byref(h)))
    return GpuIndex(h)


def build_index_sampled(dataset, train_ids, params: IndexParams = IndexParams(), device: int = 0) -> GpuIndex:
    """Config 5's sampled build (include/suco_b200.h: suco_gpu_build_index_sampled): k-means on the
    rows `train_ids` (strictly ascending) only, then every row assigned to its nearest centroid
    (kmeans.cpp:19-33) and the IMI built over all of them (index.cpp:69-96)."""
    ptr, n, d, _keep = _rows(dataset)
    tr = np.asarray(train_ids)
    if tr.ndim != 1 or (tr.size and (tr.min() < 0 or tr.max() > 0xFFFFFFFF)):
        raise ContractError("training ids must be a 1-D array of row ids")
    tr = np.ascontiguousarray(tr, np.uint32)
    h = C.c_void_p()
    ip = params._c()
    _check(_c.build_index_sampled(ptr, n, d, C.byref(ip), _p(tr, _c.u32p), tr.size, device, C.byref(h)))
    return GpuIndex(h)


def load_index(blob: bytes, dataset, device: int = 0) -> GpuIndex:
    """deserialize_index (index.cpp:191-293) + check_compatible (index.cpp:295-305), uploaded to the GPU."""
    if isinstance(blob, str):
        with open(blob, "rb") as f:
            blob = f.read()
    v = _values(dataset)
    buf = np.frombuffer(blob, np.uint8)
    h = C.c_void_p()
    _check(_c.load_index(_p(buf, _c.u8p), len(blob), _p(v, _c.f32p), v.shape[0], v.shape[1], device, C.byref(h)))
    return GpuIndex(h)


# ------------------------------------------------------------------ vecs I/O (io.hpp:15-40)
VECS_KINDS = {"fvecs": 0, "f32": 0, "bvecs": 1, "u8": 1, "ivecs": 2, "i32": 2}


def _kind(kind) -> int:
    if isinstance(kind, str):
        if kind not in VECS_KINDS:
            raise ContractError(f"unknown vecs kind {kind!r}")
        return VECS_KINDS[kind]
    return int(kind)


def _limit(limit: Optional[int]) -> int:
    return 0xFFFFFFFFFFFFFFFF if limit is None else int(limit)


def read_vecs(path: str, kind="fvecs", limit: Optional[int] = None) -> np.ndarray:
    """read_vecs (io.hpp:22-33, io.cpp:99-137): n x d float32 (bvecs / ivecs widened)."""
    k = _kind(kind)
    n, d = C.c_uint64(), C.c_uint32()
    _check(_c.read_vecs(path.encode(), k, _limit(limit), None, 0, C.byref(n), C.byref(d)))
    out = np.empty((n.value, d.value), np.float32)
    _check(_c.read_vecs(path.encode(), k, _limit(limit), _p(out, _c.f32p), n.value, C.byref(n), C.byref(d)))
    return out


def write_vecs(path: str, kind, values) -> None:
    """write_vecs (io.hpp:35-40): the inverse of read_vecs."""
    v = np.ascontiguousarray(values, np.float32)
    if v.ndim != 2:
        raise ContractError("write_vecs: values must be an n x d matrix")
    _check(_c.write_vecs(path.encode(), _kind(kind), v.shape[0], v.shape[1], _p(v, _c.f32p)))


def build_index_from_vecs(path: str, kind="fvecs", params: IndexParams = IndexParams(), limit: Optional[int] = None,
                          device: int = 0) -> GpuIndex:
    """build_index over a vecs file streamed straight into device memory (pinned, chunked)."""
    h = C.c_void_p()
    ip = params._c()
    _check(_c.build_index_from_vecs(path.encode(), _kind(kind), _limit(limit), C.byref(ip), device, C.byref(h)))
    return GpuIndex(h)


def load_index_from_vecs(blob: bytes, path: str, kind="fvecs", limit: Optional[int] = None,
                         device: int = 0) -> GpuIndex:
    """load_index with the dataset streamed from a vecs file into device memory."""
    if isinstance(blob, str):
        with open(blob, "rb") as f:
            blob = f.read()
    buf = np.frombuffer(blob, np.uint8)
    h = C.c_void_p()
    _check(_c.load_index_from_vecs(_p(buf, _c.u8p), len(blob), path.encode(), _kind(kind), _limit(limit), device,
                                   C.byref(h)))
    return GpuIndex(h)


def knn_query(index: GpuIndex, dataset, query, params: CollisionParams) -> List[Neighbor]:
    """knn_query (query.hpp:93-96) for one query; the index owns the dataset rows on the device,
    `dataset` is checked for compatibility (index.cpp:295-305) like the reference."""
    v = _values(dataset)
    n, d, _ = index.info()
    if v.shape[0] != n:
        raise IncompatibilityError(f"index was built from n = {n} points but dataset has n = {v.shape[0]}")
    if v.shape[1] != d:
        raise IncompatibilityError(f"index was built for d = {d} but dataset has d = {v.shape[1]}")
    ids, dists = index.knn_query_batch(_f32(query).reshape(1, -1), params)
    return [Neighbor(int(i), float(x)) for i, x in zip(ids[0], dists[0])]


def centroid_distances(half_query, centroids, k_half: int):
    """query.cpp:42-64: (dists true-Euclidean fp64, order by (dist, id))."""
    q = _f32(half_query).ravel()
    c = _f32(centroids).ravel()
    if k_half >= 1 and q.size and c.size != k_half * q.size:
        raise ContractError("centroid matrix does not match k_half x half dim")
    dists = np.empty(max(k_half, 1), np.float64)
    order = np.empty(max(k_half, 1), np.uint32)
    _check(_c.centroid_distances(_p(q, _c.f32p), q.size, _p(c, _c.f32p), k_half, _p(dists, _c.f64p),
                                 _p(order, _c.u32p)))
    return dists[:k_half], order[:k_half]


def dynamic_activation(alpha: float, n: int, cd1, cd2, imi_offsets) -> List[RetrievedCell]:
    """query.cpp:66-121 over the IMI given by its CSR offsets; cd = (dists, order)."""
    d1, o1 = (np.ascontiguousarray(cd1[0], np.float64), np.ascontiguousarray(cd1[1], np.uint32))
    d2, o2 = (np.ascontiguousarray(cd2[0], np.float64), np.ascontiguousarray(cd2[1], np.uint32))
    off = np.ascontiguousarray(imi_offsets, np.uint64)
    k = int(round((off.size - 1) ** 0.5))
    if k * k + 1 != off.size:
        raise ContractError("imi offsets must hold k_half^2 + 1 entries")
    if d1.size != k or o1.size != k or d2.size != k or o2.size != k:
        raise ContractError("centroid distance arrays do not match the imi's k_half")
    cap = k * k
    c1 = np.empty(cap, np.uint32)
    c2 = np.empty(cap, np.uint32)
    cum = np.empty(cap, np.uint64)
    sums = np.empty(cap, np.float64)
    cnt = C.c_uint64()
    _check(_c.dynamic_activation(alpha, n, _p(d1, _c.f64p), _p(o1, _c.u32p), _p(d2, _c.f64p), _p(o2, _c.u32p), k,
                                 _p(off, _c.u64p), _p(c1, _c.u32p), _p(c2, _c.u32p), _p(cum, _c.u64p),
                                 _p(sums, _c.f64p), cap, C.byref(cnt)))
    return [RetrievedCell(int(c1[i]), int(c2[i]), int(cum[i]), float(sums[i])) for i in range(cnt.value)]


def rerank(dataset, query, candidates, k: int) -> List[Neighbor]:
    """query.cpp:159-197: exact top-k of the candidates by (distance, id)."""
    v = _values(dataset)
    q = _f32(query).ravel()
    cands = np.ascontiguousarray(candidates, np.uint32)
    ids = np.empty(max(k, 1), np.uint32)
    dists = np.empty(max(k, 1), np.float64)
    _check(_c.rerank(_p(v, _c.f32p), v.shape[0], v.shape[1], _p(q, _c.f32p), q.size, _p(cands, _c.u32p), cands.size,
                     k, _p(ids, _c.u32p), _p(dists, _c.f64p)))
    return [Neighbor(int(i), float(x)) for i, x in zip(ids[:k], dists[:k])]


def kmeans(points, k: int, iterations: int, seed: int, device: int = 0):
    """kmeans (kmeans.cpp:118-194): dict(centroids k x dim, assignments n, repaired)."""
    pts = _f32(points)
    if pts.ndim == 1:
        pts = pts[:, None]
    n, dim = pts.shape
    cent = np.empty((max(k, 1), dim), np.float32)
    assign = np.empty(n, np.uint32)
    rep = np.empty(max(k * max(iterations, 1), 1), np.uint32)
    nrep = C.c_uint32()
    _check(_c.kmeans(_p(pts, _c.f32p), n, dim, k, iterations, seed, device, _p(cent, _c.f32p), _p(assign, _c.u32p),
                     _p(rep, _c.u32p), C.byref(nrep)))
    return dict(centroids=cent[:k], assignments=assign, repaired=rep[: nrep.value].copy())


def build_imi(first, second, k_half: int):
    """build_imi (index.cpp:69-96): (offsets k_half^2+1 u64, ids n u32)."""
    a = np.ascontiguousarray(first, np.uint32)
    b = np.ascontiguousarray(second, np.uint32)
    if a.size != b.size:
        raise ContractError(f"assignment arrays differ in length: {a.size} vs {b.size}")
    off = np.empty(max(k_half, 1) ** 2 + 1, np.uint64)
    ids = np.empty(a.size, np.uint32)
    _check(_c.build_imi(_p(a, _c.u32p), _p(b, _c.u32p), a.size, k_half, _p(off, _c.u64p), _p(ids, _c.u32p)))
    return off, ids


# ------------------------------------------------------------------ evaluation (host arithmetic)
def recall(result_ids, truth_ids, k: int) -> float:
    """|result ids ∩ exact top-k ids| / k (eval.hpp:33, eval.cpp:64-79); one query's rows."""
    if k < 1:
        raise ContractError("recall: k must be >= 1")
    truth_ids = np.asarray(truth_ids).ravel()
    result_ids = np.asarray(result_ids).ravel()
    if truth_ids.size < k:
        raise ContractError("recall: ground truth has fewer than k entries")
    if result_ids.size > k:
        raise ContractError("recall: result holds more than k entries")
    return float(np.isin(result_ids, truth_ids[:k]).sum()) / float(k)


def mre(result_dists, truth_dists, k: int) -> float:
    """Mean over ranks of (result - truth) / truth for the first k entries, ranks with a zero true
    distance dropped; all dropped -> 0 if the result is 0 there, +inf otherwise (eval.cpp:81-102)."""
    if k < 1:
        raise ContractError("mre: k must be >= 1")
    r = np.asarray(result_dists, np.float64).ravel()
    t = np.asarray(truth_dists, np.float64).ravel()
    if t.size < k or r.size < k:
        raise ContractError("mre: both lists must hold at least k entries")
    total, included, clean = 0.0, 0, True
    for i in range(k):  # in rank order, like the reference's accumulation
        if t[i] == 0.0:
            clean &= r[i] == 0.0
            continue
        total += (r[i] - t[i]) / t[i]
        included += 1
    if included:
        return total / included
    return 0.0 if clean else float("inf")
