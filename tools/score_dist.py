"""Score distribution at cfg2 (debug tool): per query, #points with score >= t and the threshold T."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench_data
import paper_2411_14754_b200 as suco
cfg = bench_data.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
base, qs = bench_data.generate(cfg)
idx = suco.build_index(base, suco.IndexParams(cfg.num_subspaces, cfg.k_half, cfg.iterations, 42), device=0)
cp = suco.CollisionParams(cfg.alpha, cfg.beta, cfg.k)
m = suco.candidate_count(cfg.beta, len(base), cfg.k)
rows = []
for i in range(int(os.environ.get("NQ", "50"))):
    sc, cands, cps, cum = idx.query_intermediates(qs[i], cp)
    ge = [int((sc >= t).sum()) for t in range(cfg.num_subspaces + 1)]
    T = max([t for t in range(1, cfg.num_subspaces + 1) if ge[t] >= m] or [0])
    rows.append((T, ge))
Ts = [r[0] for r in rows]
print("m", m, "T histogram", np.bincount(Ts, minlength=cfg.num_subspaces + 1).tolist())
for T, ge in rows[:12]:
    print(T, ge)
ratio = [ge[T - 1] / m if T >= 1 else float('nan') for T, ge in rows]
print("count(>=T-1)/m: median %.1f max %.1f" % (np.nanmedian(ratio), np.nanmax(ratio)))
ratio2 = [ge[T] / m for T, ge in rows]
print("count(>=T)/m: median %.2f max %.2f" % (np.median(ratio2), np.max(ratio2)))
