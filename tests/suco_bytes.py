"""Test helper: parse a `.suco` blob (index.cpp:147-170 — 44-byte header, layout, then per
subspace centroids_first, centroids_second, IMI offsets, IMI ids) into numpy arrays."""
from __future__ import annotations

import struct

import numpy as np


def parse(blob: bytes) -> dict:
    assert blob[:4] == b"SUCO"
    version, n, d, ns, k_half, iters, seed, mode = struct.unpack_from("<IQIIIIQI", blob, 4)
    pos = 44
    dims = []
    for _ in range(ns):
        (cnt,) = struct.unpack_from("<I", blob, pos)
        pos += 4
        dims.append(np.frombuffer(blob, np.uint32, cnt, pos).copy())
        pos += 4 * cnt
    K = k_half * k_half
    subs = []
    for s in range(ns):
        h1 = len(dims[s]) // 2  # half_split (subspace.cpp:41)
        h2 = len(dims[s]) - h1
        c1 = np.frombuffer(blob, np.float32, k_half * h1, pos).reshape(k_half, h1).copy()
        pos += 4 * k_half * h1
        c2 = np.frombuffer(blob, np.float32, k_half * h2, pos).reshape(k_half, h2).copy()
        pos += 4 * k_half * h2
        off = np.frombuffer(blob, np.uint64, K + 1, pos).copy()
        pos += 8 * (K + 1)
        ids = np.frombuffer(blob, np.uint32, n, pos).copy()
        pos += 4 * n
        subs.append({"cent1": c1, "cent2": c2, "offsets": off, "ids": ids})
    assert pos == len(blob)
    return {"version": version, "n": n, "d": d, "ns": ns, "k_half": k_half, "iters": iters, "seed": seed,
            "mode": mode, "dims": dims, "subspaces": subs}


def cell_of(sub: dict, n: int) -> np.ndarray:
    """Per point, the IMI cell holding it."""
    off = sub["offsets"].astype(np.int64)
    cells = np.repeat(np.arange(len(off) - 1, dtype=np.int64), np.diff(off))
    out = np.empty(n, np.int64)
    out[sub["ids"]] = cells
    return out
