"""Where e2e time goes at cfg2: device step vs host-buffer step vs the copies alone."""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench_data  # noqa: E402
import paper_2411_14754_b200 as suco  # noqa: E402
from paper_2411_14754_b200 import _capi  # noqa: E402

cfg = bench_data.CONFIGS["cfg2"]
base, queries = bench_data.generate(cfg)
idx = suco.build_index(base, suco.IndexParams(8, 50, 10, 42))
cp = suco.CollisionParams(cfg.alpha, cfg.beta, cfg.k)
nq, d, k = len(queries), cfg.d, cfg.k
st = torch.cuda.Stream()
idx.set_stream(st.cuda_stream)
dq = torch.from_numpy(queries).cuda()
di = torch.empty((nq, k), dtype=torch.int32, device="cuda")
dd = torch.empty((nq, k), dtype=torch.float64, device="cuda")
hq = torch.from_numpy(queries).pin_memory()
hi = torch.empty((nq, k), dtype=torch.int32).pin_memory()
hd = torch.empty((nq, k), dtype=torch.float64).pin_memory()
cpc = cp._c()


def dev():
    idx.knn_query_batch_device(dq.data_ptr(), nq, d, cp, di.data_ptr(), dd.data_ptr(), st.cuda_stream)


def host():
    rc = _capi.knn_query_batch(idx.handle, C.cast(hq.data_ptr(), _capi.f32p), nq, d, C.byref(cpc),
                               C.cast(hi.data_ptr(), _capi.u32p), C.cast(hd.data_ptr(), _capi.f64p))
    assert rc == 0


def copies():
    with torch.cuda.stream(st):
        dq.copy_(hq, non_blocking=True)
        hi.copy_(di, non_blocking=True)
        hd.copy_(dd, non_blocking=True)


def timed(fn, reps=10):
    fn()
    st.synchronize()
    ev = []
    wall = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.synchronize()
        t = time.perf_counter()
        e0.record(st)
        fn()
        e1.record(st)
        e1.synchronize()
        wall.append((time.perf_counter() - t) * 1e3)
        ev.append(e0.elapsed_time(e1))
    return np.median(ev), np.median(wall)


for name, fn in (("device step", dev), ("host-buffer step", host), ("copies only (H2D 5.1 MB + D2H 1.2 MB)", copies)):
    e, w = timed(fn)
    print(f"{name}: events {e:.3f} ms, wall {w:.3f} ms")
