"""Phase timing of the shard protocol at G = 1 (debug tool, not a bench number)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench_data  # noqa: E402
import paper_2411_14754_b200 as suco  # noqa: E402
from paper_2411_14754_b200 import candidate_count  # noqa: E402
from paper_2411_14754_b200.sharded import GpuShard, merge_topk, plan_for_shard  # noqa: E402

cfg = bench_data.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
base, queries = bench_data.generate(cfg)
idx = suco.build_index(base, suco.IndexParams(cfg.num_subspaces, cfg.k_half, cfg.iterations, 42), device=0)
G = int(os.environ.get("G", "1"))
engs = [GpuShard(idx, r, G, None) for r in range(G)]
print("block", engs[0].block, "nblocks", [e.nblocks for e in engs], flush=True)
cp = suco.CollisionParams(cfg.alpha, cfg.beta, cfg.k)
dq = torch.from_numpy(queries).cuda()
m = candidate_count(cp.beta, engs[0].n_global, cp.k)
for it in range(3):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    torch.cuda.synchronize()
    t0 = time.time()
    ev[0].record()
    hists = [e.histograms(dq, cp) for e in engs]
    ev[1].record()
    plans = [plan_for_shard(hists, r, m) for r in range(G)]
    ev[2].record()
    tops = [e.topk(dq, cp, plans[r]) for r, e in enumerate(engs)]
    ev[3].record()
    ids, dd = merge_topk([t[0] for t in tops], [t[1] for t in tops], cp.k)
    ev[4].record()
    torch.cuda.synchronize()
    print(f"iter {it}: wall {1e3 * (time.time() - t0):.1f} ms; hist {ev[0].elapsed_time(ev[1]):.2f} plan "
          f"{ev[1].elapsed_time(ev[2]):.2f} topk {ev[2].elapsed_time(ev[3]):.2f} merge {ev[3].elapsed_time(ev[4]):.2f}"
          f" stride {plans[0].stride}", flush=True)
want = idx.knn_query_batch(queries, cp)
print("parity", np.array_equal(ids.cpu().numpy().astype(np.uint32), want[0]), np.array_equal(dd.cpu().numpy(), want[1]))

if os.environ.get("COMM"):
    import torch.distributed as dist
    from paper_2411_14754_b200.sharded import TorchComm, knn_query_distributed
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    comm = TorchComm()
    stream = torch.cuda.Stream()
    for it in range(4):
        torch.cuda.synchronize()
        t0 = time.time()
        with torch.cuda.stream(stream):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ids, dd = knn_query_distributed(engs[0], comm, dq, cp)
            e1.record(stream)
        e1.synchronize()
        print(f"comm iter {it}: wall {1e3 * (time.time() - t0):.1f} ms, events {e0.elapsed_time(e1):.2f} ms", flush=True)
    # the same with profiler-free host timing per phase
    with torch.cuda.stream(stream):
        for it in range(2):
            torch.cuda.synchronize()
            t = [time.time()]
            hist = engs[0].histograms(dq, cp); torch.cuda.synchronize(); t.append(time.time())
            hists = comm.allgather_var(hist); torch.cuda.synchronize(); t.append(time.time())
            plan = plan_for_shard(hists, 0, m); torch.cuda.synchronize(); t.append(time.time())
            i2, s2 = engs[0].topk(dq, cp, plan); torch.cuda.synchronize(); t.append(time.time())
            a = comm.allgather_var(i2); b = comm.allgather_var(s2); torch.cuda.synchronize(); t.append(time.time())
            merge_topk(a, b, cp.k); torch.cuda.synchronize(); t.append(time.time())
            print("phases ms:", [round(1e3 * (y - x), 2) for x, y in zip(t, t[1:])], flush=True)
    dist.destroy_process_group()
