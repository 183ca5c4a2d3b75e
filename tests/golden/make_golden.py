"""Generates the golden fixtures in tests/golden/ by running the REFERENCE itself.

Run here (where /root/reference exists and oracle/_ref/libsuco_ref.so is
built from its sources):  python tests/golden/make_golden.py
Every array below is the output of the unmodified reference library
(oracle/_ref, compiled from /root/reference/proj/src by oracle/Makefile)
through its public API; the fixtures pin both the C restatement and the GPU
path on machines where the reference is absent.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import ref  # noqa: E402


def corpus(R):
    """Descriptor-style corpus like acceptance.cpp:70-74, scaled down: sift_like + hold-out."""
    full = R.clustered(2100, 32, 16, 7, 20.0, 140.0, 18.0, True)
    base, queries = R.hold_out(full, 100, 8)
    return base, queries


def main():
    R = ref()
    out = {}
    # --- end-to-end: build + knn_query at three parameter points
    base, queries = corpus(R)
    idx = R.build_index(base, 4, 12, 5, 42, 0, 0)
    blob = np.frombuffer(idx.serialize(), np.uint8)
    res = {}
    for tag, (a, b, k) in {"p0": (0.05, 0.05, 10), "p1": (0.1, 0.02, 40), "p2": (0.02, 0.005, 5)}.items():
        ids, dists, _ = idx.knn_query_batch(base, queries, a, b, k, threads=1)
        res[f"{tag}_ids"] = ids
        res[f"{tag}_dists"] = dists
        res[f"{tag}_params"] = np.array([a, b, k], np.float64)
    scores, cands, cps, cum = idx.query_intermediates(base, queries[0], 0.05, 0.05, 10)
    np.savez_compressed(os.path.join(HERE, "e2e_small.npz"), base=base, queries=queries, index=blob,
                        scores_q0=scores, cands_q0=cands, cells_q0=cps, cum_q0=cum, **res)

    # --- shuffled layout, d % 4 != 0, odd subspace split
    data = R.clustered(600, 22, 6, 77, 0.0, 50.0, 4.0, False)
    qs = R.uniform(20, 22, 78, 0.0, 50.0)
    idx2 = R.build_index(data, 3, 7, 4, 9, 1, 0)
    ids2, d2, _ = idx2.knn_query_batch(data, qs, 0.1, 0.05, 7, threads=1)
    np.savez_compressed(os.path.join(HERE, "e2e_shuffled.npz"), base=data, queries=qs,
                        index=np.frombuffer(idx2.serialize(), np.uint8), ids=ids2, dists=d2,
                        params=np.array([0.1, 0.05, 7], np.float64))

    # --- traversal: random IMIs / centroid distances (test_query.cpp:105-152 style)
    g = R.rng(2024)
    trav = {}
    i = 0
    for k_half in (1, 2, 3, 5, 8, 17, 64):
        for quantize in (False, True):
            for alpha in (0.01, 0.1, 0.5, 1.0):
                n = 1 + g.uniform_below(400)
                d1, o1 = g.centroid_distances(k_half, quantize)
                dd2, o2 = g.centroid_distances(k_half, quantize)
                off, ids = g.imi(k_half, n)
                c1, c2, cum, sums = R.traverse(0, alpha, n, d1, o1, dd2, o2, k_half, off, ids)
                trav[f"t{i}_meta"] = np.array([k_half, n, alpha], np.float64)
                trav[f"t{i}_d1"], trav[f"t{i}_o1"], trav[f"t{i}_d2"], trav[f"t{i}_o2"] = d1, o1, dd2, o2
                trav[f"t{i}_off"] = off
                trav[f"t{i}_c1"], trav[f"t{i}_c2"], trav[f"t{i}_cum"], trav[f"t{i}_sums"] = c1, c2, cum, sums
                i += 1
    trav["count"] = np.array([i])
    np.savez_compressed(os.path.join(HERE, "traversal.npz"), **trav)

    # --- centroid distances incl. ties (test_query.cpp:53-69) and a random block
    cent = R.uniform(50, 8, 5, 0.0, 10.0)
    q = R.uniform(1, 8, 6, 0.0, 10.0)[0]
    dd, oo = R.centroid_distances(q, cent, 50)
    np.savez_compressed(os.path.join(HERE, "centroid_distances.npz"), cent=cent, q=q, dists=dd, order=oo)

    # --- rerank (test_query.cpp:188-214 shape) and k-means (test_kmeans.cpp:70-83 shape)
    data = R.uniform(200, 12, 9)
    qq = R.uniform(3, 12, 10)
    cand = np.arange(200, dtype=np.uint32)[::5].copy()
    rr = {f"ids{j}": R.rerank(data, qq[j], cand, 15)[0] for j in range(3)}
    rr.update({f"dists{j}": R.rerank(data, qq[j], cand, 15)[1] for j in range(3)})
    np.savez_compressed(os.path.join(HERE, "rerank.npz"), data=data, queries=qq, cands=cand, **rr)

    pts = R.uniform(1000, 6, 31)
    km = R.kmeans(pts, 20, 8, 5, threads=1)
    dup = np.array([[0.0, 0.0] if i % 2 == 0 else [50.0, 50.0] for i in range(64)], np.float32)
    km2 = R.kmeans(dup, 8, 5, 13, threads=1)
    np.savez_compressed(os.path.join(HERE, "kmeans.npz"), pts=pts, centroids=km["centroids"],
                        assignments=km["assignments"], repaired=km["repaired"], dup=dup,
                        dup_centroids=km2["centroids"], dup_assignments=km2["assignments"],
                        dup_repaired=km2["repaired"])
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
