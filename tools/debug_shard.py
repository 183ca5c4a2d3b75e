import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2411_14754_b200 as suco
from paper_2411_14754_b200 import sharded as S
from oracle.oracle import oracle
O = oracle()
full = O.clustered(20050, 32, 40, 78, 20, 140, 18, True)
base, qs = O.hold_out(full, 50, 78)
idx = suco.build_index(base, suco.IndexParams(4, 16, 3, 42))
cp = suco.CollisionParams(0.05, 0.005, 10)
want_i, want_d = idx.knn_query_batch(qs, cp)
for G, blk in ((1, 4096), (2, 512)):
    sh = [S.GpuShard(idx, r, G, blk) for r in range(G)]
    print('G', G, [(s.n_local, s.nblocks, s.block) for s in sh])
    q = torch.from_numpy(qs).cuda()
    hists = [s.histograms(q, cp) for s in sh]
    torch.cuda.synchronize()
    m = suco.candidate_count(cp.beta, idx.n, cp.k)
    tot = sum(h.to(torch.int64).sum(dim=1) for h in hists)
    print(' m', m, 'total_ge q0', tot[0].tolist())
    s0, c0, _, _ = idx.query_intermediates(qs[0], cp)
    print(' ref ge q0', [int((s0 >= t).sum()) for t in range(6)])
    for r, s in enumerate(sh):
        plan = S.plan_for_shard(hists, r, m)
        print(' plan', r, 'T', plan.T[:4].tolist(), 'counts', plan.counts[:4].tolist(), 'stride', plan.stride)
        ids = torch.full((q.shape[0], cp.k), -7, dtype=torch.int32, device='cuda')
        sq = torch.full((q.shape[0], cp.k), -1.0, dtype=torch.float64, device='cuda')
        rc = S._c.shard_topk(s.index.handle, S.C.c_void_p(q.data_ptr()), q.shape[0], s.d, S.C.byref(cp._c()),
                             S.C.c_void_p(plan.T.data_ptr()), S.C.c_void_p(plan.quota.data_ptr()),
                             S.C.c_void_p(plan.base.data_ptr()), S.C.c_void_p(plan.counts.data_ptr()), plan.stride,
                             S.C.c_void_p(ids.data_ptr()), S.C.c_void_p(sq.data_ptr()),
                             S.C.c_void_p(torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        print('  rc', rc, S._c.last_error(), 'ids q0', ids[0].tolist(), 'sq', sq[0, :3].tolist())
    ids, dd = S.emulate(sh, q, cp)
    print(' emulate equal', np.array_equal(ids.cpu().numpy().astype(np.uint32), want_i), np.array_equal(dd.cpu().numpy(), want_d))
    print(' want q0', want_i[0].tolist())
