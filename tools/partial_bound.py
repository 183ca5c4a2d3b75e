"""Experiment: how many re-rank candidates a partial-dimension lower bound would rule out.
For sampled queries of a config: the candidate set (query_intermediates), each candidate's exact
squared distance D, the partial sum over the first h dims (a lower bound of D), and tau = the
k-th smallest D. Prints the fraction of candidates with partial(h) > tau for several h."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench_data
import paper_2411_14754_b200 as suco

cfg = bench_data.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg4"]
base, qs = bench_data.generate(cfg)
idx = suco.build_index(base, suco.IndexParams(cfg.num_subspaces, cfg.k_half, cfg.iterations, 42), device=0)
cp = suco.CollisionParams(cfg.alpha, cfg.beta, cfg.k)
hs = sorted({4, 8, 12, 16, 48, 96, cfg.d // 4, cfg.d // 2} - {0})
fr = {h: [] for h in hs}
for i in range(0, len(qs), len(qs) // 20):
    _, cands, _, _ = idx.query_intermediates(qs[i], cp)
    X = base[cands].astype(np.float64)
    diff2 = (X - qs[i].astype(np.float64)) ** 2
    D = diff2.sum(1)
    tau = np.sort(D)[cfg.k - 1]
    for h in hs:
        fr[h].append(float((diff2[:, :h].sum(1) > tau).mean()))
    print(i, "m", len(cands), "tau %.4g median D %.4g" % (tau, np.median(D)),
          {h: round(fr[h][-1], 3) for h in hs}, flush=True)
print("mean pruned fraction by h:", {h: round(float(np.mean(v)), 3) for h, v in fr.items()})
