"""Seeded synthetic inputs for the five BASELINE.json configs (benchmark input prep only).

The reference measures on real corpora that are not in this container
(SIFT/GIST/Deep); per SURVEY §8(d) seeded Gaussian mixtures
with each config's shape, value range and spread stand in for them. This is
NOT the reference generator (that one is a single mt19937_64 stream, too slow
for 10^7-10^8 points); it is a chunked numpy PCG64 mixture with the same
recipe: component means U[lo, hi]^d, isotropic sigma, optional u8
quantisation (round + clip to 0..255) or L2 normalisation. cfg1-cfg3: n + Q
points drawn from one mixture, Q of them held out (seeded, without
replacement) as queries, base and queries both in ascending original-id order
(io.cpp:212-252). cfg4/cfg5 (the point-sharded configs): one PCG64 stream
per 2,048-row chunk, so any rank generates exactly its own block-cyclic rows
(generate_shard) and all chunks generate in parallel; queries are their own
stream of the same mixture. Both the GPU path and the reference CPU path
consume the same arrays.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Tuple

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    d: int
    clusters: int
    lo: float
    hi: float
    sigma: float
    quantize: bool
    normalize: bool
    queries: int
    num_subspaces: int
    k_half: int
    alpha: float
    beta: float
    k: int
    seed: int
    iterations: int = 10
    train_sample: float = 1.0  # cfg5: k-means trained on a 1% sample
    parallel: bool = False     # cfg4/cfg5: chunk-seeded streams (per-rank rows, all host cores)

    def describe(self) -> str:
        kind = "u8-valued" if self.quantize else ("unit-norm" if self.normalize else "float32")
        return (f"{self.name}: n={self.n:,} d={self.d} {kind} {self.clusters}-component mixture, "
                f"{self.queries:,} queries, N_s={self.num_subspaces}, {self.k_half}x{self.k_half} centroids, "
                f"alpha={self.alpha} beta={self.beta} k={self.k}")


CONFIGS = {
    "cfg1": Config("cfg1", 100_000, 128, 100, 0.0, 100.0, 10.0, False, False, 1_000, 8, 50, 0.05, 0.005, 10, 1001),
    "cfg2": Config("cfg2", 1_000_000, 128, 1000, 20.0, 140.0, 18.0, True, False, 10_000, 8, 50, 0.05, 0.005, 10, 1002),
    "cfg3": Config("cfg3", 1_000_000, 960, 1000, 0.0, 1.0, 0.05, False, False, 1_000, 16, 50, 0.05, 0.01, 10, 1003),
    "cfg4": Config("cfg4", 10_000_000, 96, 10_000, -1.0, 1.0, 0.2, False, True, 10_000, 8, 64, 0.03, 0.005, 10, 1004,
                   parallel=True),
    "cfg5": Config("cfg5", 100_000_000, 128, 100_000, 20.0, 140.0, 18.0, True, False, 10_000, 8, 100, 0.02, 0.002,
                   10, 1005, train_sample=0.01, parallel=True),
}


def train_ids(cfg: Config, n: int) -> np.ndarray:
    """The seeded training sample of a sampled build (cfg5: 1 % of the rows), ascending u32 ids."""
    size = max(cfg.k_half, int(round(n * cfg.train_sample)))
    if size >= n:
        return np.arange(n, dtype=np.uint32)
    rng = np.random.default_rng(cfg.seed + 7)
    return np.sort(rng.choice(n, size=size, replace=False)).astype(np.uint32)


CHUNK = 2048  # rows per seeded stream (divides every shard block size)


def _mixture(cfg: Config):
    return np.random.default_rng(cfg.seed).uniform(cfg.lo, cfg.hi, size=(cfg.clusters, cfg.d)).astype(np.float32)


def _fill(cfg: Config, centers, out, lo, hi, key):
    g = np.random.default_rng(np.random.SeedSequence([cfg.seed, key]))
    v = g.standard_normal((hi - lo, cfg.d), dtype=np.float32)
    v *= np.float32(cfg.sigma)
    v += centers[g.integers(0, cfg.clusters, size=hi - lo)]
    if cfg.quantize:
        np.clip(np.rint(v, out=v), 0.0, 255.0, out=v)
    if cfg.normalize:
        v /= np.sqrt(np.einsum("ij,ij->i", v, v))[:, None]
    out[:] = v


def _chunks(cfg: Config, n: int, chunk_ids, out: np.ndarray):
    """Chunks chunk_ids (rows [c * CHUNK, (c + 1) * CHUNK) of the base) into `out`, back to back,
    on all host cores."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    centers = _mixture(cfg)
    starts, pos = [], 0
    for c in chunk_ids:
        rows = min(n, (c + 1) * CHUNK) - c * CHUNK
        starts.append((c, pos, rows))
        pos += rows
    with ThreadPoolExecutor(os.cpu_count() or 1) as ex:
        list(ex.map(lambda t: _fill(cfg, centers, out[t[1]:t[1] + t[2]], t[0] * CHUNK, t[0] * CHUNK + t[2], t[0]),
                    starts))
    return pos


def _queries(cfg: Config, nq: int) -> np.ndarray:
    q = np.empty((nq, cfg.d), np.float32)
    _fill(cfg, _mixture(cfg), q, 0, nq, 1 << 32)
    return q


def _generate_parallel(cfg: Config, n: int, nq: int) -> Tuple[np.ndarray, np.ndarray]:
    base = np.empty((n, cfg.d), np.float32)
    _chunks(cfg, n, range((n + CHUNK - 1) // CHUNK), base)
    return base, _queries(cfg, nq)


def generate_shard(cfg: Config, block: int, num_shards: int, shard: int, n: int | None = None,
                   queries: int | None = None) -> Tuple[np.ndarray, np.ndarray]:
    """(shard `shard`'s rows — global blocks j = shard mod G of `block` ids, in id order —,
    all queries) of a chunk-seeded config, without materialising the other shards' rows."""
    if not cfg.parallel or block % CHUNK:
        raise ValueError("per-shard generation needs a chunk-seeded config and block % 2048 == 0")
    n = cfg.n if n is None else n
    nq = cfg.queries if queries is None else queries
    nb = (n + block - 1) // block
    per = block // CHUNK
    chunk_ids = [j * per + i for j in range(shard, nb, num_shards) for i in range(per) if (j * per + i) * CHUNK < n]
    rows = sum(min(n, (c + 1) * CHUNK) - c * CHUNK for c in chunk_ids)
    out = np.empty((rows, cfg.d), np.float32)
    _chunks(cfg, n, chunk_ids, out)
    return out, _queries(cfg, nq)


def generate(cfg: Config, n: int | None = None, queries: int | None = None,
             chunk: int = 1 << 17) -> Tuple[np.ndarray, np.ndarray]:
    """(base n x d float32, queries Q x d float32) for `cfg` (optionally resized for tests)."""
    n = cfg.n if n is None else n
    nq = cfg.queries if queries is None else queries
    if cfg.parallel:
        return _generate_parallel(cfg, n, nq)
    total = n + nq
    rng = np.random.default_rng(cfg.seed)
    centers = rng.uniform(cfg.lo, cfg.hi, size=(cfg.clusters, cfg.d))
    labels = rng.integers(0, cfg.clusters, size=total)
    out = np.empty((total, cfg.d), np.float32)
    for lo in range(0, total, chunk):
        hi = min(total, lo + chunk)
        v = centers[labels[lo:hi]] + cfg.sigma * rng.standard_normal((hi - lo, cfg.d))
        if cfg.quantize:
            np.clip(np.rint(v, out=v), 0.0, 255.0, out=v)
        if cfg.normalize:
            v /= np.sqrt(np.einsum("ij,ij->i", v, v))[:, None]
        out[lo:hi] = v
    held = np.zeros(total, bool)
    held[rng.choice(total, size=nq, replace=False)] = True
    return np.ascontiguousarray(out[~held]), np.ascontiguousarray(out[held])
