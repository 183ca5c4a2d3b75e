"""Where the index build time goes: upload vs device build (python tools/build_phases.py cfg4)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench_data  # noqa: E402
import paper_2411_14754_b200 as suco  # noqa: E402

cfg = bench_data.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg4"]
base, _ = bench_data.generate(cfg, queries=8)
p = suco.IndexParams(cfg.num_subspaces, cfg.k_half, cfg.iterations, 42)
train = bench_data.train_ids(cfg, len(base)) if cfg.train_sample < 1 else None


def build(x):
    return suco.build_index_sampled(x, train, p) if train is not None else suco.build_index(x, p)


torch.cuda.synchronize()
t = time.time(); dev = torch.from_numpy(base).cuda(); torch.cuda.synchronize(); up = time.time() - t
t = time.time(); i1 = build(dev); torch.cuda.synchronize(); bd = time.time() - t
del i1
t = time.time(); i2 = build(base); torch.cuda.synchronize(); bh = time.time() - t
print(f"{cfg.name}: torch pageable upload {up:.2f} s ({base.nbytes / up / 1e9:.1f} GB/s); build from device rows {bd:.2f} s; "
      f"build from host rows {bh:.2f} s")
