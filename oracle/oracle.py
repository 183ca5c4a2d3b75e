"""TEST INFRASTRUCTURE ONLY — numpy/ctypes front-end over the two CPU checkers.

* ``Oracle``: the plain-C restatement, oracle/_build/libsuco_oracle.so
  (oracle/suco_oracle.c, every function citing the reference file:line).
* ``Ref``: the UNMODIFIED reference library compiled from its own sources,
  oracle/_ref/libsuco_ref.so (oracle/ref_harness.cpp is only glue).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module, and only as the checker / CPU baseline — the
product path (paper_2411_14754_b200) never touches it.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libsuco_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsuco_ref.so")

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
f32p = C.POINTER(C.c_float)
f64p = C.POINTER(C.c_double)


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def build_if_needed():
    import subprocess

    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    if os.path.isdir("/root/reference/proj"):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


@dataclass
class Layout:
    dims: np.ndarray  # concatenated per-subspace dims
    sizes: np.ndarray
    split: np.ndarray

    def half_dims(self, s: int, half: int) -> np.ndarray:
        start = int(self.sizes[:s].sum())
        sz, sp = int(self.sizes[s]), int(self.split[s])
        d = self.dims[start:start + sz]
        return d[:sp] if half == 0 else d[sp:]


class _Lib:
    prefix = ""
    path = ""

    def __init__(self):
        if not os.path.exists(self.path):
            raise FileNotFoundError(f"{self.path} missing; run `make -C oracle`")
        self.lib = C.CDLL(self.path)
        self._err = getattr(self.lib, self.prefix + "last_error")
        self._err.restype = C.c_char_p

    def _fn(self, name, restype=C.c_int):
        f = getattr(self.lib, self.prefix + name)
        f.restype = restype
        return f

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self._err().decode())


class Oracle(_Lib):
    """The C restatement (oracle/suco_oracle.c)."""

    prefix = "so_"
    path = ORACLE_SO

    def splitmix64(self, x):
        return self._fn("splitmix64", C.c_uint64)(C.c_uint64(x))

    def derive_seed(self, s, t):
        return self._fn("derive_seed", C.c_uint64)(C.c_uint64(s), C.c_uint64(t))

    def fnv1a(self, b: bytes, seed=0xCBF29CE484222325):
        return self._fn("fnv1a", C.c_uint64)(C.c_char_p(b), C.c_uint64(len(b)), C.c_uint64(seed))

    def collision_count(self, alpha, n):
        return self._fn("collision_count", C.c_uint64)(C.c_double(alpha), C.c_uint64(n))

    def candidate_count(self, beta, n, k):
        return self._fn("candidate_count", C.c_uint64)(C.c_double(beta), C.c_uint64(n), C.c_uint64(k))

    def validate_params(self, alpha, beta, k, n):
        self._check(self._fn("validate_params")(C.c_double(alpha), C.c_double(beta), C.c_uint32(k), C.c_uint64(n)))

    def clustered(self, n, d, clusters, seed, lo, hi, sigma, quantize):
        out = np.empty((n, d), np.float32)
        self._check(self._fn("clustered")(C.c_uint64(n), C.c_uint32(d), C.c_uint32(clusters), C.c_uint64(seed),
                                          C.c_double(lo), C.c_double(hi), C.c_double(sigma), C.c_int(int(quantize)),
                                          _p(out, f32p)))
        return out

    def uniform(self, n, d, seed, lo=0.0, hi=1.0):
        out = np.empty((n, d), np.float32)
        self._check(self._fn("uniform")(C.c_uint64(n), C.c_uint32(d), C.c_uint64(seed), C.c_float(lo), C.c_float(hi),
                                        _p(out, f32p)))
        return out

    def hold_out(self, data: np.ndarray, count, seed):
        data = np.ascontiguousarray(data, np.float32)
        n, d = data.shape
        base = np.empty((n - count, d), np.float32) if count < n else np.empty((0, d), np.float32)
        q = np.empty((count, d), np.float32)
        self._check(self._fn("hold_out")(_p(data, f32p), C.c_uint64(n), C.c_uint32(d), C.c_uint64(count),
                                         C.c_uint64(seed), _p(base, f32p), _p(q, f32p)))
        return base, q

    def sample_subspaces(self, d, ns, mode, seed) -> Layout:
        dims = np.empty(d, np.uint32)
        sizes = np.empty(max(ns, 1), np.uint32)
        split = np.empty(max(ns, 1), np.uint32)
        self._check(self._fn("sample_subspaces")(C.c_uint32(d), C.c_uint32(ns), C.c_uint32(mode), C.c_uint64(seed),
                                                 _p(dims, u32p), _p(sizes, u32p), _p(split, u32p)))
        return Layout(dims, sizes, split)

    def sqdist4(self, a, b):
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        return self._fn("sqdist4", C.c_double)(_p(a, f32p), _p(b, f32p), C.c_size_t(a.size))

    def kmeans(self, points, k, iters, seed, with_wcss=False):
        points = np.ascontiguousarray(points, np.float32)
        n, dim = points.shape
        cent = np.empty((k, dim), np.float32)
        assign = np.empty(n, np.uint32)
        rep = np.empty(max(k * iters, 1), np.uint32)
        nrep = np.zeros(1, np.uint32)
        wcss = np.empty(iters, np.float64)
        self._check(self._fn("kmeans")(_p(points, f32p), C.c_uint64(n), C.c_uint32(dim), C.c_uint32(k),
                                       C.c_uint32(iters), C.c_uint64(seed), _p(cent, f32p), _p(assign, u32p),
                                       _p(rep, u32p), _p(nrep, u32p), _p(wcss, f64p) if with_wcss else None))
        out = dict(centroids=cent, assignments=assign, repaired=rep[: int(nrep[0])].copy())
        if with_wcss:
            out["wcss"] = wcss
        return out

    def build_imi(self, first, second, k_half):
        first = np.ascontiguousarray(first, np.uint32)
        second = np.ascontiguousarray(second, np.uint32)
        if first.size != second.size:
            raise OracleError(5, "assignment arrays differ in length")
        offsets = np.empty(k_half * k_half + 1, np.uint64)
        ids = np.empty(first.size, np.uint32)
        self._check(self._fn("build_imi")(_p(first, u32p), _p(second, u32p), C.c_uint64(first.size),
                                          C.c_uint32(k_half), _p(offsets, u64p), _p(ids, u32p)))
        return offsets, ids

    # ---- index
    def build_index(self, data, ns, k_half, iters, seed, mode=0, threads=0) -> "OracleIndex":
        data = np.ascontiguousarray(data, np.float32)
        h = C.c_void_p()
        self._check(self._fn("build_index")(_p(data, f32p), C.c_uint64(data.shape[0]), C.c_uint32(data.shape[1]),
                                            C.c_uint32(ns), C.c_uint32(k_half), C.c_uint32(iters), C.c_uint64(seed),
                                            C.c_uint32(mode), C.c_uint(threads), C.byref(h)))
        return OracleIndex(self, h)

    def build_index_sampled(self, data, train_ids, ns, k_half, iters, seed, mode=0, threads=0) -> "OracleIndex":
        """Config 5's sampled build (suco_oracle.h: so_build_index_sampled)."""
        data = np.ascontiguousarray(data, np.float32)
        train = np.ascontiguousarray(train_ids, np.uint32)
        h = C.c_void_p()
        self._check(self._fn("build_index_sampled")(
            _p(data, f32p), C.c_uint64(data.shape[0]), C.c_uint32(data.shape[1]), C.c_uint32(ns), C.c_uint32(k_half),
            C.c_uint32(iters), C.c_uint64(seed), C.c_uint32(mode), _p(train, u32p), C.c_uint64(train.size),
            C.c_uint(threads), C.byref(h)))
        return OracleIndex(self, h)

    def load_index(self, blob: bytes) -> "OracleIndex":
        h = C.c_void_p()
        buf = np.frombuffer(blob, np.uint8)
        self._check(self._fn("deserialize_index")(_p(buf, u8p), C.c_uint64(len(blob)), C.byref(h)))
        return OracleIndex(self, h)

    # ---- query stages
    def centroid_distances(self, half_query, centroids, k_half):
        q = np.ascontiguousarray(half_query, np.float32)
        c = np.ascontiguousarray(centroids, np.float32)
        dists = np.empty(k_half, np.float64)
        order = np.empty(k_half, np.uint32)
        self._check(self._fn("centroid_distances")(_p(q, f32p), C.c_uint32(q.size), _p(c, f32p), C.c_uint32(k_half),
                                                   _p(dists, f64p), _p(order, u32p)))
        return dists, order

    def traverse(self, kind, alpha, n, d1, o1, d2, o2, k_half, offsets):
        cap = k_half * k_half
        c1 = np.empty(cap, np.uint32)
        c2 = np.empty(cap, np.uint32)
        cum = np.empty(cap, np.uint64)
        sums = np.empty(cap, np.float64)
        cnt = C.c_uint64()
        args = [np.ascontiguousarray(x, t) for x, t in
                ((d1, np.float64), (o1, np.uint32), (d2, np.float64), (o2, np.uint32), (offsets, np.uint64))]
        self._check(self._fn("traverse")(C.c_int(kind), C.c_double(alpha), C.c_uint64(n), _p(args[0], f64p),
                                         _p(args[1], u32p), _p(args[2], f64p), _p(args[3], u32p), C.c_uint32(k_half),
                                         _p(args[4], u64p), _p(c1, u32p), _p(c2, u32p), _p(cum, u64p),
                                         _p(sums, f64p), C.c_uint64(cap), C.byref(cnt)))
        m = cnt.value
        return c1[:m].copy(), c2[:m].copy(), cum[:m].copy(), sums[:m].copy()

    def rerank(self, data, query, cands, k):
        data = np.ascontiguousarray(data, np.float32)
        q = np.ascontiguousarray(query, np.float32)
        cands = np.ascontiguousarray(cands, np.uint32)
        ids = np.empty(max(k, 1), np.uint32)
        dists = np.empty(max(k, 1), np.float64)
        cnt = C.c_uint32()
        self._check(self._fn("rerank")(_p(data, f32p), C.c_uint64(data.shape[0]), C.c_uint32(data.shape[1]),
                                       _p(q, f32p), C.c_uint32(q.size), _p(cands, u32p), C.c_uint64(cands.size),
                                       C.c_uint32(k), _p(ids, u32p), _p(dists, f64p), C.byref(cnt)))
        return ids[: cnt.value].copy(), dists[: cnt.value].copy()


class OracleIndex:
    def __init__(self, lib: _Lib, handle):
        self.lib = lib
        self.h = handle

    def __del__(self):
        try:
            self.lib._fn("index_free", None)(self.h)
        except Exception:
            pass

    def info(self):
        n = C.c_uint64()
        d = C.c_uint32()
        ns = C.c_uint32()
        kh = C.c_uint32()
        self.lib._fn("index_info")(self.h, C.byref(n), C.byref(d), C.byref(ns), C.byref(kh))
        return n.value, d.value, ns.value, kh.value

    def serialize(self) -> bytes:
        ln = C.c_uint64()
        self.lib._check(self.lib._fn("serialize_index")(self.h, None, C.c_uint64(0), C.byref(ln)))
        buf = np.empty(ln.value, np.uint8)
        self.lib._check(self.lib._fn("serialize_index")(self.h, _p(buf, u8p), C.c_uint64(ln.value), C.byref(ln)))
        return buf.tobytes()

    def knn_query_batch(self, data, queries, alpha, beta, k, threads=0):
        data = np.ascontiguousarray(data, np.float32)
        queries = np.ascontiguousarray(queries, np.float32)
        nq, qlen = queries.shape
        ids = np.zeros((nq, k), np.uint32)
        dists = np.zeros((nq, k), np.float64)
        counts = np.zeros(nq, np.uint32)
        wall = C.c_double()
        self.lib._check(self.lib._fn("knn_query_batch")(
            self.h, _p(data, f32p), C.c_uint64(data.shape[0]), C.c_uint32(data.shape[1]), _p(queries, f32p),
            C.c_uint64(nq), C.c_uint32(qlen), C.c_double(alpha), C.c_double(beta), C.c_uint32(k),
            C.c_uint(threads or (os.cpu_count() or 1)), _p(ids, u32p), _p(dists, f64p), _p(counts, u32p),
            C.byref(wall)))
        return ids, dists, wall.value

    def query_intermediates(self, data, query, alpha, beta, k):
        data = np.ascontiguousarray(data, np.float32)
        q = np.ascontiguousarray(query, np.float32)
        n, d = data.shape
        _, _, ns, _ = self.info()
        scores = np.empty(n, np.uint32)
        cands = np.empty(n, np.uint32)
        m = C.c_uint64()
        cps = np.empty(ns, np.uint32)
        cum = np.empty(ns, np.uint64)
        self.lib._check(self.lib._fn("query_intermediates")(
            self.h, _p(data, f32p), C.c_uint64(n), C.c_uint32(d), _p(q, f32p), C.c_uint32(q.size),
            C.c_double(alpha), C.c_double(beta), C.c_uint32(k), _p(scores, u32p), _p(cands, u32p), C.byref(m),
            _p(cps, u32p), _p(cum, u64p)))
        return scores, cands[: m.value].copy(), cps, cum


class Ref(_Lib):
    """The reference library itself (oracle/_ref/libsuco_ref.so)."""

    prefix = "ref_"
    path = REF_SO

    def splitmix64(self, x):
        return self._fn("splitmix64", C.c_uint64)(C.c_uint64(x))

    def derive_seed(self, s, t):
        return self._fn("derive_seed", C.c_uint64)(C.c_uint64(s), C.c_uint64(t))

    def fnv1a(self, b: bytes, seed=0xCBF29CE484222325):
        return self._fn("fnv1a", C.c_uint64)(C.c_char_p(b), C.c_uint64(len(b)), C.c_uint64(seed))

    def collision_count(self, alpha, n):
        return self._fn("collision_count", C.c_uint64)(C.c_double(alpha), C.c_uint64(n))

    def candidate_count(self, beta, n, k):
        return self._fn("candidate_count", C.c_uint64)(C.c_double(beta), C.c_uint64(n), C.c_uint64(k))

    def validate_params(self, alpha, beta, k, n):
        self._check(self._fn("validate_params")(C.c_double(alpha), C.c_double(beta), C.c_uint32(k), C.c_uint64(n)))

    def clustered(self, n, d, clusters, seed, lo, hi, sigma, quantize):
        out = np.empty((n, d), np.float32)
        self._check(self._fn("clustered")(C.c_uint64(n), C.c_uint32(d), C.c_uint32(clusters), C.c_uint64(seed),
                                          C.c_double(lo), C.c_double(hi), C.c_double(sigma), C.c_int(int(quantize)),
                                          _p(out, f32p)))
        return out

    def uniform(self, n, d, seed, lo=0.0, hi=1.0):
        out = np.empty((n, d), np.float32)
        self._check(self._fn("uniform")(C.c_uint64(n), C.c_uint32(d), C.c_uint64(seed), C.c_float(lo), C.c_float(hi),
                                        _p(out, f32p)))
        return out

    def hold_out(self, data, count, seed):
        data = np.ascontiguousarray(data, np.float32)
        n, d = data.shape
        base = np.empty((max(n - count, 0), d), np.float32)
        q = np.empty((count, d), np.float32)
        self._check(self._fn("hold_out")(_p(data, f32p), C.c_uint64(n), C.c_uint32(d), C.c_uint64(count),
                                         C.c_uint64(seed), _p(base, f32p), _p(q, f32p)))
        return base, q

    def sample_subspaces(self, d, ns, mode, seed) -> Layout:
        dims = np.empty(d, np.uint32)
        sizes = np.empty(max(ns, 1), np.uint32)
        split = np.empty(max(ns, 1), np.uint32)
        self._check(self._fn("sample_subspaces")(C.c_uint32(d), C.c_uint32(ns), C.c_uint32(mode), C.c_uint64(seed),
                                                 _p(dims, u32p), _p(sizes, u32p), _p(split, u32p)))
        return Layout(dims, sizes, split)

    def kmeans(self, points, k, iters, seed, threads=1, with_wcss=False):
        points = np.ascontiguousarray(points, np.float32)
        n, dim = points.shape
        cent = np.empty((k, dim), np.float32)
        assign = np.empty(n, np.uint32)
        rep = np.empty(max(k * iters, 1), np.uint32)
        nrep = np.zeros(1, np.uint32)
        wcss = np.empty(iters, np.float64)
        self._check(self._fn("kmeans")(_p(points, f32p), C.c_uint64(n), C.c_uint32(dim), C.c_uint32(k),
                                       C.c_uint32(iters), C.c_uint64(seed), C.c_uint(threads), _p(cent, f32p),
                                       _p(assign, u32p), _p(rep, u32p), _p(nrep, u32p),
                                       _p(wcss, f64p) if with_wcss else None))
        out = dict(centroids=cent, assignments=assign, repaired=rep[: int(nrep[0])].copy())
        if with_wcss:
            out["wcss"] = wcss
        return out

    def build_imi(self, first, second, k_half):
        first = np.ascontiguousarray(first, np.uint32)
        second = np.ascontiguousarray(second, np.uint32)
        offsets = np.empty(k_half * k_half + 1, np.uint64)
        ids = np.empty(first.size, np.uint32)
        self._check(self._fn("build_imi")(_p(first, u32p), _p(second, u32p), C.c_uint64(first.size),
                                          C.c_uint32(k_half), _p(offsets, u64p), _p(ids, u32p)))
        return offsets, ids

    def build_index(self, data, ns, k_half, iters, seed, mode=0, threads=0) -> "RefIndex":
        data = np.ascontiguousarray(data, np.float32)
        h = C.c_void_p()
        self._check(self._fn("build_index")(_p(data, f32p), C.c_uint64(data.shape[0]), C.c_uint32(data.shape[1]),
                                            C.c_uint32(ns), C.c_uint32(k_half), C.c_uint32(iters), C.c_uint64(seed),
                                            C.c_uint32(mode), C.c_uint(threads), C.byref(h)))
        return RefIndex(self, h)

    def load_index(self, blob: bytes) -> "RefIndex":
        h = C.c_void_p()
        buf = np.frombuffer(blob, np.uint8)
        self._check(self._fn("index_from_bytes")(_p(buf, u8p), C.c_uint64(len(blob)), C.byref(h)))
        return RefIndex(self, h)

    def centroid_distances(self, half_query, centroids, k_half):
        q = np.ascontiguousarray(half_query, np.float32)
        c = np.ascontiguousarray(centroids, np.float32)
        dists = np.empty(k_half, np.float64)
        order = np.empty(k_half, np.uint32)
        self._check(self._fn("centroid_distances")(_p(q, f32p), C.c_uint32(q.size), _p(c, f32p), C.c_uint32(k_half),
                                                   _p(dists, f64p), _p(order, u32p)))
        return dists, order

    def traverse(self, kind, alpha, n, d1, o1, d2, o2, k_half, offsets, ids):
        cap = k_half * k_half
        c1 = np.empty(cap, np.uint32)
        c2 = np.empty(cap, np.uint32)
        cum = np.empty(cap, np.uint64)
        sums = np.empty(cap, np.float64)
        cnt = C.c_uint64()
        a = [np.ascontiguousarray(x, t) for x, t in
             ((d1, np.float64), (o1, np.uint32), (d2, np.float64), (o2, np.uint32), (offsets, np.uint64),
              (ids, np.uint32))]
        self._check(self._fn("traverse")(C.c_int(kind), C.c_double(alpha), C.c_uint64(n), _p(a[0], f64p),
                                         _p(a[1], u32p), _p(a[2], f64p), _p(a[3], u32p), C.c_uint32(k_half),
                                         _p(a[4], u64p), _p(a[5], u32p), _p(c1, u32p), _p(c2, u32p), _p(cum, u64p),
                                         _p(sums, f64p), C.c_uint64(cap), C.byref(cnt)))
        m = cnt.value
        return c1[:m].copy(), c2[:m].copy(), cum[:m].copy(), sums[:m].copy()

    def rerank(self, data, query, cands, k):
        data = np.ascontiguousarray(data, np.float32)
        q = np.ascontiguousarray(query, np.float32)
        cands = np.ascontiguousarray(cands, np.uint32)
        ids = np.empty(max(k, 1), np.uint32)
        dists = np.empty(max(k, 1), np.float64)
        cnt = C.c_uint32()
        self._check(self._fn("rerank")(_p(data, f32p), C.c_uint64(data.shape[0]), C.c_uint32(data.shape[1]),
                                       _p(q, f32p), C.c_uint32(q.size), _p(cands, u32p), C.c_uint64(cands.size),
                                       C.c_uint32(k), _p(ids, u32p), _p(dists, f64p), C.byref(cnt)))
        return ids[: cnt.value].copy(), dists[: cnt.value].copy()

    def exact_knn(self, data, query, k):
        data = np.ascontiguousarray(data, np.float32)
        q = np.ascontiguousarray(query, np.float32)
        ids = np.empty(k, np.uint32)
        dists = np.empty(k, np.float64)
        self._check(self._fn("exact_knn")(_p(data, f32p), C.c_uint64(data.shape[0]), C.c_uint32(data.shape[1]),
                                          _p(q, f32p), C.c_uint32(k), _p(ids, u32p), _p(dists, f64p)))
        return ids, dists

    def hardware_threads(self):
        return self._fn("hardware_threads", C.c_uint)()

    def rng(self, seed) -> "RefRng":
        return RefRng(self, seed)


class RefRng:
    """A std::mt19937_64 living inside the reference library (for testsupport fakes)."""

    def __init__(self, lib: Ref, seed):
        self.lib = lib
        f = lib._fn("rng_new", C.c_void_p)
        f.argtypes = [C.c_uint64]
        self.h = C.c_void_p(f(seed))

    def __del__(self):
        try:
            self.lib._fn("rng_free", None)(self.h)
        except Exception:
            pass

    def uniform_below(self, bound):
        return self.lib._fn("rng_uniform_below", C.c_uint64)(self.h, C.c_uint64(bound))

    def uniform_unit(self):
        return self.lib._fn("rng_uniform_unit", C.c_double)(self.h)

    def centroid_distances(self, k_half, quantize):
        d = np.empty(k_half, np.float64)
        o = np.empty(k_half, np.uint32)
        self.lib._check(self.lib._fn("rng_centroid_distances")(self.h, C.c_uint32(k_half), C.c_int(int(quantize)),
                                                               _p(d, f64p), _p(o, u32p)))
        return d, o

    def imi(self, k_half, n):
        off = np.empty(k_half * k_half + 1, np.uint64)
        ids = np.empty(n, np.uint32)
        self.lib._check(self.lib._fn("rng_imi")(self.h, C.c_uint32(k_half), C.c_uint64(n), _p(off, u64p),
                                                _p(ids, u32p)))
        return off, ids


class RefIndex:
    def __init__(self, lib: Ref, handle):
        self.lib = lib
        self.h = handle
        self._ds = None
        self._ds_key = None

    def __del__(self):
        try:
            self.lib._fn("index_free", None)(self.h)
            if self._ds is not None:
                self.lib._fn("dataset_free", None)(self._ds)
        except Exception:
            pass

    def info(self):
        n = C.c_uint64()
        d = C.c_uint32()
        ns = C.c_uint32()
        kh = C.c_uint32()
        self.lib._fn("index_info")(self.h, C.byref(n), C.byref(d), C.byref(ns), C.byref(kh))
        return n.value, d.value, ns.value, kh.value

    def serialize(self) -> bytes:
        ln = C.c_uint64()
        self.lib._check(self.lib._fn("index_serialize")(self.h, None, C.c_uint64(0), C.byref(ln)))
        buf = np.empty(ln.value, np.uint8)
        self.lib._check(self.lib._fn("index_serialize")(self.h, _p(buf, u8p), C.c_uint64(ln.value), C.byref(ln)))
        return buf.tobytes()

    def subspace(self, si, h1, h2):
        n, d, ns, kh = self.info()
        c1 = np.empty((kh, h1), np.float32)
        c2 = np.empty((kh, h2), np.float32)
        off = np.empty(kh * kh + 1, np.uint64)
        ids = np.empty(n, np.uint32)
        self.lib._check(self.lib._fn("index_subspace")(self.h, C.c_uint32(si), _p(c1, f32p), _p(c2, f32p),
                                                       _p(off, u64p), _p(ids, u32p)))
        return c1, c2, off, ids

    def _dataset(self, data):
        key = (data.ctypes.data, data.shape)
        if self._ds is None or self._ds_key != key:
            if self._ds is not None:
                self.lib._fn("dataset_free", None)(self._ds)
            h = C.c_void_p()
            self.lib._check(self.lib._fn("dataset_new")(_p(data, f32p), C.c_uint64(data.shape[0]),
                                                        C.c_uint32(data.shape[1]), C.byref(h)))
            self._ds, self._ds_key, self._ds_ref = h, key, data
        return self._ds

    def knn_query_batch(self, data, queries, alpha, beta, k, threads=0, traversal=0):
        data = np.ascontiguousarray(data, np.float32)
        queries = np.ascontiguousarray(queries, np.float32)
        ds = self._dataset(data)
        nq, qlen = queries.shape
        ids = np.zeros((nq, k), np.uint32)
        dists = np.zeros((nq, k), np.float64)
        counts = np.zeros(nq, np.uint32)
        wall = C.c_double()
        self.lib._check(self.lib._fn("knn_query_batch")(
            self.h, ds, _p(queries, f32p), C.c_uint64(nq), C.c_uint32(qlen), C.c_double(alpha), C.c_double(beta),
            C.c_uint32(k), C.c_int(traversal), C.c_uint(threads), _p(ids, u32p), _p(dists, f64p), _p(counts, u32p),
            C.byref(wall)))
        return ids, dists, wall.value

    def sc_scores(self, data, query, alpha):
        """compute_sc_scores (sc_linear.hpp:45) over this index's layout."""
        data = np.ascontiguousarray(data, np.float32)
        ds = self._dataset(data)
        q = np.ascontiguousarray(query, np.float32)
        scores = np.empty(data.shape[0], np.uint32)
        self.lib._check(self.lib._fn("sc_scores")(self.h, ds, _p(q, f32p), C.c_uint32(q.size), C.c_double(alpha),
                                                  _p(scores, u32p)))
        return scores

    def sc_linear_query(self, data, query, alpha, beta, k):
        """sc_linear_query (sc_linear.hpp:52) over this index's layout -> (ids, dists)."""
        data = np.ascontiguousarray(data, np.float32)
        ds = self._dataset(data)
        q = np.ascontiguousarray(query, np.float32)
        ids = np.empty(k, np.uint32)
        dists = np.empty(k, np.float64)
        cnt = C.c_uint32()
        self.lib._check(self.lib._fn("sc_linear_query")(self.h, ds, _p(q, f32p), C.c_uint32(q.size), C.c_double(alpha),
                                                        C.c_double(beta), C.c_uint32(k), _p(ids, u32p),
                                                        _p(dists, f64p), C.byref(cnt)))
        return ids[: cnt.value].copy(), dists[: cnt.value].copy()

    def query_intermediates(self, data, query, alpha, beta, k):
        data = np.ascontiguousarray(data, np.float32)
        ds = self._dataset(data)
        q = np.ascontiguousarray(query, np.float32)
        n = data.shape[0]
        _, _, ns, _ = self.info()
        scores = np.empty(n, np.uint32)
        cands = np.empty(n, np.uint32)
        m = C.c_uint64()
        cps = np.empty(ns, np.uint32)
        cum = np.empty(ns, np.uint64)
        self.lib._check(self.lib._fn("query_intermediates")(
            self.h, ds, _p(q, f32p), C.c_uint32(q.size), C.c_double(alpha), C.c_double(beta), C.c_uint32(k),
            _p(scores, u32p), _p(cands, u32p), C.byref(m), _p(cps, u32p), _p(cum, u64p)))
        return scores, cands[: m.value].copy(), cps, cum


_oracle = None
_ref = None


def oracle() -> Oracle:
    global _oracle
    if _oracle is None:
        _oracle = Oracle()
    return _oracle


def ref() -> Ref:
    global _ref
    if _ref is None:
        _ref = Ref()
    return _ref


def ref_available() -> bool:
    return os.path.exists(REF_SO)
