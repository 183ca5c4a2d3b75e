// C-ABI, the multi-GPU shard protocol; the reference is single
// host, so this is the sharded form of build_index (index.cpp:98-145) and
// knn_query (query.cpp:199-262), bit-identical to them for any shard count.
//
// Points are split block-cyclically: global block j = ids [j*b, (j+1)*b)
// lives on shard j % G (b a multiple of the dense select's 2048-id pieces).
// Every shard keeps the layout, all centroids and the GLOBAL cell sizes, so
// its traversal makes the global Dynamic-Activation cut; it scores only its
// own points. Per query tile (one stream, collectives enqueued on it):
//   traverse -> K1 piece histograms -> totals #(score >= t)
//   == allgather totals ==  -> T, need = m - #(score > T); ties at T per block
//   == allgather block ties == -> quotas in GLOBAL id order (the reference's
//   (score desc, id asc) top-m, query.cpp:242-260) -> K3 local candidates
//   -> exact local re-rank: top-min(k, count) (squared distance, global id)
//   == allgather local top-k == -> G-way merge by (distance, id), sqrt
//   (query.cpp:181-192).
// Exchange volume per query: 64 B + 4 B x ceil(#blocks / G) + 12 B x k per
// shard (cfg4 at G = 8, b = 8,192: about 1.0 KB, i.e. ~10 MB per 10K-query
// tile per shard).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "build.h"
#include "capi_internal.h"
#include "comm.h"

using namespace suco_gpu;

namespace {

uint64_t shard_rows(uint64_t n, uint32_t b, uint32_t G, uint32_t r) {
    const uint64_t nb = (n + b - 1) / b;
    uint64_t rows = 0;
    for (uint64_t j = r; j < nb; j += G) rows += std::min<uint64_t>(b, n - j * b);
    return rows;
}

void check_block(uint32_t block) {
    if (block < kDensePiece || block % kDensePiece != 0) {
        raise(SUCO_ERR_CONFIG, "shard block size must be a positive multiple of " + std::to_string(kDensePiece) +
                                   " ids (the dense select's pieces), got " + std::to_string(block));
    }
}

// The shard's select tables; the sharded select is the dense one.
void finalize_shard(suco_gpu_index* x) {
    finalize_dense(x, true);
    if (!x->dense) {
        raise(SUCO_ERR_CONFIG, "sharded queries need the dense select (N_s <= 16 with the cell masks in shared memory)");
    }
    set_l2_persisting(x);
}

// The protocol's select as ONE scoring pass (dense.cu, "the shard protocol's single pass"): the
// sampled totals are summed over the shards so every shard takes the same speculative bound L and
// tie cut, the fused pass scores the shard's pieces once, #(score > L) is summed and the per-block
// ties gathered, and the plan cuts the reference's global top-m exactly. Returns false — after
// every shard agreed on it — when any shard flagged a query (T != L, a quota past the cut, an
// overflowing buffer); the caller then runs the two-pass protocol for the tile.
bool shard_fused_select(const suco_gpu_index* x, suco_gpu_query_ctx* c, suco_gpu_query_ctx::Slot& sl, suco_comm* comm,
                        uint64_t nt, uint64_t m, uint32_t G, uint32_t r, uint64_t nb, uint32_t nbl, uint32_t nbl_max,
                        cudaStream_t s) {
    const HostIndex& h = x->host;
    const Tuning& tn = x->tune;
    if (!x->dense || nt == 0) return false;
    DenseArgs da = dense_args(x, sl, nt);
    da.m = m;
    // pieces: the unsharded path's choice over the shard's points, dividing the id block
    uint32_t wp = tn.dense_piece ? tn.dense_piece : fused_piece(h.n, nt, da.half ? 16u : 32u);
    while (wp > kDensePiece && x->block % wp) wp /= 2;
    if (x->block % wp) return false;
    da.WP = wp;
    da.P = static_cast<uint32_t>((h.n + wp - 1) / wp);
    const uint32_t ppbf = x->block / wp;
    const uint32_t P_global = static_cast<uint32_t>((x->n_global + wp - 1) / wp);
    da.shG = G;
    da.shR = r;
    da.shPPB = ppbf;
    const uint32_t P2 = static_cast<uint32_t>((h.n + kDensePiece - 1) / kDensePiece);
    da.sWP = kDensePiece;
    da.pstride = P2 <= 64 ? 1u : std::min<uint32_t>(64, P2 / 16);
    da.Ps = (P2 + da.pstride - 1) / da.pstride;
    sl.dsample.reserve(nt * da.Ps * 8 * da.nc);
    da.hsample = sl.dsample.p;
    const uint64_t fit = (1ull << 30) / (2ull * nt * da.P) / 8 * 8;
    const uint64_t minb = uint64_t(kDenseBuf) * (da.WP / kDensePiece);
    da.B = static_cast<uint32_t>(std::min<uint64_t>(da.WP, std::max<uint64_t>(minb, fit)));
    if (tn.dense_buf) da.B = tn.dense_buf;
    sl.dcbuf.reserve(nt * da.P * da.B);
    sl.dccnt.reserve(nt * da.P);
    sl.dL.reserve(nt);
    sl.dh2.reserve(nt * da.P);
    sl.dT.reserve(nt);
    sl.dquota.reserve(nt * da.P);
    sl.dbase.reserve(2 * nt * da.P);
    sl.dflag.reserve(5 * nt + 3);
    da.cbuf = sl.dcbuf.p;
    da.ccnt = sl.dccnt.p;
    da.L = sl.dL.p;
    da.h2 = sl.dh2.p;
    da.T = sl.dT.p;
    da.quota = sl.dquota.p;
    da.base = sl.dbase.p;
    da.base2 = sl.dbase.p + nt * da.P;
    da.qflag = sl.dflag.p;
    da.pcut = sl.dflag.p + 2 * nt + 1;
    da.clist = sl.dflag.p + 3 * nt + 1;
    da.nclist = sl.dflag.p + 5 * nt + 1;
    da.stage_all = tn.dense_stage;
    da.no_cut = tn.dense_nocut;
    da.compact_mode = tn.dense_compact;
    da.compact_rows = tn.dense_compact_rows;
    da.cands = sl.cands.p;
    c->sh_s17.reserve(nt * 17);
    c->sh_gt.reserve(nt);
    c->sh_gts.reserve(nt);
    c->sh_nflag.reserve(1);
    c->sh_ties.reserve(nt * nbl_max);
    c->sh_ties_all.reserve(G * nt * nbl_max);
    c->sh_qblk.reserve(nt * nbl_max);
    // S0: the same L and tie cut on every shard
    CUDA_TRY(launch_shard_sample(da, c->sh_s17.p, s));
    comm->allreduce_sum_u32(c->sh_s17.p, nt * 17, s);
    CUDA_TRY(launch_shard_bound(da, c->sh_s17.p, x->n_global, P_global, s));
    // S1: one scoring pass over the shard's pieces
    CUDA_TRY(launch_dense_fused_pass(da, s));
    // S2: #(score > L) summed, the blocks' ties gathered
    CUDA_TRY(launch_shard_fused_sums(da, ppbf, nbl, nbl_max, c->sh_gt.p, c->sh_ties.p, s));
    CUDA_TRY(cudaMemcpyAsync(c->sh_gts.p, c->sh_gt.p, nt * 4, cudaMemcpyDeviceToDevice, s));
    comm->allreduce_sum_u32(c->sh_gts.p, nt, s);
    comm->allgather(c->sh_ties.p, c->sh_ties_all.p, nt * nbl_max * 4, s);
    // S3: the plan; any flag on any shard sends the tile to the two-pass protocol
    CUDA_TRY(cudaMemsetAsync(c->sh_nflag.p, 0, 4, s));
    CUDA_TRY(launch_shard_fused_plan(da, c->sh_gts.p, c->sh_gt.p, c->sh_ties_all.p, G, r, nb, ppbf, nbl, nbl_max,
                                     c->sh_qblk.p, c->sh_counts.p, c->sh_nflag.p, s));
    comm->allreduce_sum_u32(c->sh_nflag.p, 1, s);
    uint32_t nflag = 0;
    CUDA_TRY(cudaMemcpyAsync(&nflag, c->sh_nflag.p, 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    c->launches += 8;
    if (tn.dense_stats)
        std::fprintf(stderr, "[suco] shard %u/%u single pass: %u flagged queries of %llu (all shards)%s\n", r, G, nflag,
                     static_cast<unsigned long long>(nt), nflag ? ": two-pass protocol for the tile" : "");
    if (nflag) return false;
    CUDA_TRY(launch_dense_compaction(da, s));
    c->launches += 2;
    return true;
}

// The protocol over one query batch (all ranks call it with the same queries and params).
void shard_run(const suco_gpu_index* x, suco_gpu_query_ctx* c, suco_comm* comm, const float* h_q, const float* d_q,
               uint64_t nq, uint32_t qlen, const suco_collision_params* p, uint32_t* d_ids, double* d_dists,
               uint32_t* h_ids, double* h_dists, cudaStream_t user) {
    const uint32_t G = static_cast<uint32_t>(comm->size), r = static_cast<uint32_t>(comm->rank);
    const uint64_t n_global = x->n_global;
    const uint32_t b = x->block, ppb = b / kDensePiece, k = p->k;
    const uint64_t nb = (n_global + b - 1) / b;
    const uint32_t nbl = r < nb ? static_cast<uint32_t>((nb - r + G - 1) / G) : 0u;
    const uint32_t nbl_max = static_cast<uint32_t>((nb + G - 1) / G);
    const uint64_t m = suco_candidate_count(p->beta, n_global, k);
    const uint64_t target = suco_collision_count(p->alpha, n_global);
    cudaStream_t s = c->pipe[0];
    CUDA_TRY(cudaEventRecord(c->ev_in, user));
    CUDA_TRY(cudaStreamWaitEvent(s, c->ev_in, 0));
    // tile: the memory budget's, agreed across ranks (every rank runs the same collectives)
    const uint64_t P = (x->host.n + kDensePiece - 1) / kDensePiece;
    const uint64_t nc = x->host.layout.ns > 8 ? 2 : 1;
    const uint64_t per = uint64_t(x->host.layout.ns) * x->K * 4 + 64 + m * 4 + (k > 32 ? m * 12 : 0) + qlen * 4 +
                         uint64_t(G) * (64 + nbl_max * 4 + k * 12) + nbl_max * 8 + P * (16 * nc + 8) + k * 12 +
                         P * (14 + 2 * kDenseBuf) + 128 * 16 * nc + G * 68 + 32;  // + the single pass's buffers
    // the tile count is agreed once per (nq, m, k) and cached (the agreement is a host round trip)
    if (c->sh_key[0] != nq || c->sh_key[1] != m || c->sh_key[2] != k || !c->sh_tiles) {
        uint64_t budget = x->tune.scratch_bytes;
        if (!budget) {
            if (!c->budget) {
                size_t free_b = 0, total_b = 0;
                CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
                c->budget = std::max<uint64_t>(64ull << 20, std::min<uint64_t>(32ull << 30, free_b / 2));
            }
            budget = c->budget;
        }
        const uint64_t fit = std::max<uint64_t>(1, budget / per);
        c->sh_tiles = agree_max(comm, (nq + fit - 1) / fit, s);
        c->sh_key[0] = nq, c->sh_key[1] = m, c->sh_key[2] = k;
    }
    const uint64_t tiles = c->sh_tiles;
    const uint64_t tile = (nq + tiles - 1) / tiles;
    begin_call(c, nq, m, s);
    const uint64_t sent0 = comm->bytes_sent;
    auto& sl = c->slot[0];
    for (uint64_t q0 = 0; q0 < nq; q0 += tile) {
        const uint64_t nt = std::min(tile, nq - q0);
        const float* tq = d_q ? d_q + q0 * qlen : nullptr;
        if (h_q) {
            sl.q.reserve(tile * qlen);
            CUDA_TRY(cudaMemcpyAsync(sl.q.p, h_q + q0 * qlen, nt * qlen * 4, cudaMemcpyHostToDevice, s));
            tq = sl.q.p;
        }
        stage_traverse(x, c, sl, tq, nt, target, s, nullptr, nullptr, true);
        c->sh_counts.reserve(nt);
        sl.cands.reserve(nt * m);
        const bool fused = x->tune.dense_fused && !(x->dense_half && x->tune.dense_pair) &&
                           shard_fused_select(x, c, sl, comm, nt, m, G, r, nb, nbl, nbl_max, s);
        if (!fused) {
        DenseArgs da = dense_args(x, sl, nt);
        da.m = m;
        sl.dhist.reserve(nt * da.P * 8 * da.nc);
        sl.dT.reserve(nt);
        sl.dquota.reserve(nt * da.P);
        sl.dbase.reserve(nt * da.P);
        da.hist = sl.dhist.p;
        da.T = sl.dT.p;
        da.quota = sl.dquota.p;
        da.base = sl.dbase.p;
        c->sh_tot.reserve(nt * 16);
        c->sh_tot_all.reserve(G * nt * 16);
        c->sh_ties.reserve(nt * nbl_max);
        c->sh_ties_all.reserve(G * nt * nbl_max);
        c->sh_need.reserve(nt);
        c->sh_qblk.reserve(nt * nbl_max);
        c->sh_counts.reserve(nt);
        sl.cands.reserve(nt * m);
        da.cands = sl.cands.p;
        // select: K1, exchange 1, ties, exchange 2, quotas, K3
        CUDA_TRY(launch_dense_hist(da, s));
        CUDA_TRY(launch_shard_totals(da, c->sh_tot.p, s));
        comm->allgather(c->sh_tot.p, c->sh_tot_all.p, nt * 16 * 4, s);
        CUDA_TRY(launch_shard_ties(da, c->sh_tot_all.p, G, ppb, nbl, nbl_max, sl.dT.p, c->sh_need.p, c->sh_ties.p, s));
        comm->allgather(c->sh_ties.p, c->sh_ties_all.p, nt * nbl_max * 4, s);
        CUDA_TRY(launch_shard_quota(da, c->sh_ties_all.p, G, r, nb, ppb, nbl, nbl_max, c->sh_need.p, c->sh_qblk.p,
                                    c->sh_counts.p, s));
        CUDA_TRY(launch_dense_emit(da, s));
        c->launches += 5;
        }
        // local exact re-rank, global ids, exchange 3, merge
        c->sh_ids.reserve(nt * k);
        c->sh_sq.reserve(nt * k);
        c->sh_ids_all.reserve(G * nt * k);
        c->sh_sq_all.reserve(G * nt * k);
        RerankArgs ra{};
        rerank_args(x, ra);
        ra.queries = tq;
        ra.cands = sl.cands.p;
        ra.m = m;
        ra.k = k;
        ra.counts = c->sh_counts.p;
        ra.squared = true;
        ra.out_ids = c->sh_ids.p;
        ra.out_dists = c->sh_sq.p;
        if (k > 32) {
            sl.all_d.reserve(nt * m);
            sl.all_id.reserve(nt * m);
            ra.all_d = sl.all_d.p;
            ra.all_id = sl.all_id.p;
        }
        CUDA_TRY(launch_rerank(ra, nt, s));
        CUDA_TRY(launch_shard_ids(c->sh_ids.p, nt * k, b, G, r, s));
        c->launches += (ra.data8 ? 2 : 1) + (k > 32 ? 1 : 0) + 1;
        comm->allgather(c->sh_ids.p, c->sh_ids_all.p, nt * k * 4, s);
        comm->allgather(c->sh_sq.p, c->sh_sq_all.p, nt * k * 8, s);
        uint32_t* oi = d_ids ? d_ids + q0 * k : nullptr;
        double* od = d_dists ? d_dists + q0 * k : nullptr;
        if (h_ids) {
            sl.out_ids.reserve(tile * k);
            sl.out_d.reserve(tile * k);
            oi = sl.out_ids.p;
            od = sl.out_d.p;
        }
        CUDA_TRY(launch_merge_topk(c->sh_ids_all.p, c->sh_sq_all.p, G, nt, k, oi, od, s));
        c->launches += 1;
        if (h_ids) {
            CUDA_TRY(cudaMemcpyAsync(h_ids + q0 * k, oi, nt * k * 4, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaMemcpyAsync(h_dists + q0 * k, od, nt * k * 8, cudaMemcpyDeviceToHost, s));
        }
    }
    c->exchange_bytes = comm->bytes_sent - sent0;
    CUDA_TRY(cudaEventRecord(c->ev_out, s));
    CUDA_TRY(cudaStreamWaitEvent(user, c->ev_out, 0));
}

void check_shard_query(const suco_gpu_index* x, const suco_comm* comm, uint32_t qlen, const suco_collision_params* p) {
    if (!x) raise(SUCO_ERR_CONTRACT, "index is null");
    if (!comm) raise(SUCO_ERR_CONTRACT, "communicator is null");
    if (static_cast<uint32_t>(comm->size) != x->num_shards || static_cast<uint32_t>(comm->rank) != x->shard) {
        raise(SUCO_ERR_CONTRACT, "communicator rank " + std::to_string(comm->rank) + " of " + std::to_string(comm->size) +
                                     " does not hold shard " + std::to_string(x->shard) + " of " +
                                     std::to_string(x->num_shards));
    }
    check_query_len(qlen, x->host.d);
    validate_params(p, x->n_global);
}

}  // namespace

extern "C" {

int suco_gpu_shard_block_hint(uint64_t n, uint32_t num_shards, uint32_t* block) {
    return guarded([&] {
        if (!block) raise(SUCO_ERR_CONTRACT, "null argument");
        if (num_shards < 1) raise(SUCO_ERR_CONFIG, "num_shards must be >= 1");
        // the quota's id span is about 0.1-0.16 n (measured); >= 16 block rounds
        // across the shards keep the tie quota from landing on one shard: b <= n / (100 G),
        // a power of two in [2048, 65536] (cfg4 at G = 8: 8,192; cfg5: 65,536)
        const uint64_t want = std::max<uint64_t>(1, n / (100ull * num_shards));
        uint32_t b = kDensePiece;
        while (b < 65536 && uint64_t(b) * 2 <= want) b *= 2;
        *block = b;
    });
}

int suco_gpu_make_shard(const suco_gpu_index* full, uint32_t shard, uint32_t num_shards, uint32_t block,
                        suco_gpu_index** out) {
    return guarded([&] {
        if (!full || !out) raise(SUCO_ERR_CONTRACT, "null argument");
        *out = nullptr;
        if (full->num_shards != 1) raise(SUCO_ERR_CONTRACT, "shards are cut from an unsharded index");
        if (num_shards < 1 || shard >= num_shards) raise(SUCO_ERR_CONFIG, "shard must be < num_shards");
        check_block(block);
        DeviceGuard g(full->device);
        const uint64_t n = full->host.n;
        const uint32_t d = full->host.d, ns = full->host.layout.ns;
        const uint64_t nb = (n + block - 1) / block;
        const uint64_t n_local = shard_rows(n, block, num_shards, shard);
        if (n_local == 0) raise(SUCO_ERR_CONFIG, "shard owns no points (n too small for this block size)");
        suco_gpu_index* x = new_index_on(full->device);
        try {
            x->tune = full->tune;
            x->host.n = n_local;
            x->host.d = d;
            x->host.p = full->host.p;
            x->host.layout = full->host.layout;
            x->host.cent1 = full->host.cent1;
            x->host.cent2 = full->host.cent2;
            x->shard = shard;
            x->num_shards = num_shards;
            x->block = block;
            x->n_global = n;
            x->data_int_max = full->data_int_max;
            x->dpad = full->dpad;
            x->qpad = full->qpad;
            x->qrec = full->qrec;
            x->qpre = full->qpre;
            x->qsplit = full->qsplit;
            // rows of the owned blocks, back to back (and their u8 / int8 copies)
            x->data.reserve(n_local * d);
            if (x->dpad) x->data8.reserve(n_local * x->dpad);
            if (x->qpad) x->q8.reserve(n_local * x->qrec);
            uint64_t lo = 0;
            for (uint64_t j = shard; j < nb; j += num_shards) {
                const uint64_t len = std::min<uint64_t>(block, n - j * block);
                CUDA_TRY(cudaMemcpyAsync(x->data.p + lo * d, full->data.p + j * block * d, len * d * 4,
                                         cudaMemcpyDeviceToDevice, x->own));
                if (x->dpad) {
                    CUDA_TRY(cudaMemcpyAsync(x->data8.p + lo * x->dpad, full->data8.p + j * block * x->dpad,
                                             len * x->dpad, cudaMemcpyDeviceToDevice, x->own));
                }
                lo += len;
            }
            if (x->qpad) {  // the int8 records of the owned rows, packed from them (a row's record depends on the row alone)
                x->q8_rows = n_local;
                CUDA_TRY(launch_pack_q8(x->data.p, n_local, d, x->qpad, x->qrec, x->qpre, x->qsplit, x->q8.p, x->own));
            }
            upload_codebooks(x);
            x->K = full->K;
            const uint64_t K = x->K;
            // GLOBAL cell sizes: every shard makes the global Dynamic-Activation cut
            x->cell_size.reserve(ns * K);
            CUDA_TRY(cudaMemcpyAsync(x->cell_size.p, full->cell_size.p, ns * K * 4, cudaMemcpyDeviceToDevice, x->own));
            // local IMI: owned ids of every cell, as local ids, ascending
            DevBuf<uint32_t> counts;
            counts.reserve(ns * K);
            CUDA_TRY(launch_shard_imi(full->ids.p, full->cell_off.p, n, ns, x->K, block, num_shards, shard, counts.p,
                                      nullptr, 0, nullptr, x->own));
            std::vector<uint32_t> hc(ns * K), hoff(ns * (K + 1));
            CUDA_TRY(cudaMemcpyAsync(hc.data(), counts.p, ns * K * 4, cudaMemcpyDeviceToHost, x->own));
            CUDA_TRY(cudaStreamSynchronize(x->own));
            for (uint32_t sub = 0; sub < ns; ++sub) {
                uint32_t run = 0;
                for (uint64_t c = 0; c < K; ++c) {
                    hoff[sub * (K + 1) + c] = run;
                    run += hc[sub * K + c];
                }
                hoff[sub * (K + 1) + K] = run;
            }
            x->cell_off.reserve(ns * (K + 1));
            CUDA_TRY(cudaMemcpyAsync(x->cell_off.p, hoff.data(), hoff.size() * 4, cudaMemcpyHostToDevice, x->own));
            x->ids.reserve(ns * n_local);
            CUDA_TRY(launch_shard_imi(full->ids.p, full->cell_off.p, n, ns, x->K, block, num_shards, shard, nullptr,
                                      x->cell_off.p, n_local, x->ids.p, x->own));
            finalize_shard(x);
        } catch (...) {
            delete x;
            throw;
        }
        *out = x;
    });
}

int suco_gpu_build_shard(const float* rows, uint64_t n_global, uint32_t d, const suco_index_params* params,
                         uint32_t block, const uint32_t* train_ids, uint64_t n_train, suco_comm* comm, int device,
                         suco_gpu_index** out) {
    return guarded([&] {
        if (!out) raise(SUCO_ERR_CONTRACT, "output handle pointer is null");
        *out = nullptr;
        if (!comm) raise(SUCO_ERR_CONTRACT, "communicator is null");
        DeviceGuard g(device);
        OwnStream os;
        const uint32_t G = static_cast<uint32_t>(comm->size), r = static_cast<uint32_t>(comm->rank);
        suco_gpu_index* x = nullptr;
        // local checks (in the reference's order), then one agreement so that an error on any rank
        // stops every rank before the first data collective
        int code = SUCO_OK;
        std::string msg;
        uint64_t n_local = 0;
        try {
            if (!params) raise(SUCO_ERR_CONTRACT, "index params are null");
            if (n_global < 1 || d < 1) raise(SUCO_ERR_CONTRACT, "dataset requires n >= 1 and d >= 1");
            check_block(block);
            n_local = shard_rows(n_global, block, G, r);
            if (n_local && !rows) raise(SUCO_ERR_CONTRACT, "shard rows are null");
            x = new_index_on(device);
            if (n_local) upload_data(x, rows, n_local, d);  // finiteness of this shard's rows (core.cpp:15-19)
            if (params->k_half < 1) raise(SUCO_ERR_CONFIG, "k_half must be >= 1");
            if (params->iterations < 1) raise(SUCO_ERR_CONFIG, "iterations must be >= 1");
            const uint64_t nfit = train_ids ? n_train : n_global;
            if (nfit < params->k_half) {
                raise(SUCO_ERR_CONFIG, std::string(train_ids ? "training sample" : "dataset") + " has n = " +
                                           std::to_string(nfit) + " points, fewer than k_half = " +
                                           std::to_string(params->k_half));
            }
            if (n_global > 0xFFFFFFFFull) raise(SUCO_ERR_CONTRACT, "dataset exceeds 32-bit point-id capacity");
            for (uint64_t i = 0; train_ids && i < n_train; ++i) {
                if (train_ids[i] >= n_global || (i && train_ids[i] <= train_ids[i - 1])) {
                    raise(SUCO_ERR_CONTRACT, "training ids must be strictly ascending and < n (entry " +
                                                 std::to_string(i) + ")");
                }
            }
            x->host.layout = sample_subspaces(d, params->num_subspaces, params->mode, params->seed);
        } catch (const Status& s) {
            code = s.code;
            msg = s.msg;
        } catch (...) {
            code = SUCO_ERR_INTERNAL;
            msg = "sharded build: setup failed (out of memory?)";
        }
        const int agreed = agree_status(comm, code, os.s);
        if (agreed != SUCO_OK) {
            delete x;
            raise(agreed, code ? msg : "the sharded build failed on another rank");
        }
        try {
            x->host.n = n_local;
            x->host.d = d;
            x->host.p = *params;
            x->shard = r;
            x->num_shards = G;
            x->block = block;
            x->n_global = n_global;
            if (!n_local) x->data.reserve(1);
            const uint32_t ns = params->num_subspaces;
            const uint64_t K = uint64_t(params->k_half) * params->k_half;
            x->K = static_cast<uint32_t>(K);
            x->cell_off.reserve(uint64_t(ns) * (K + 1));
            x->ids.reserve(uint64_t(ns) * std::max<uint64_t>(n_local, 1));
            x->cell_size.reserve(uint64_t(ns) * K);
            BuildOutputs bo{x->cell_off.p, x->ids.p, &x->host.cent1, &x->host.cent2};
            build_shard_device(x->data.p, n_local, n_global, d, block, x->host.layout, *params, comm, bo,
                               x->cell_size.p, x->own, x->tune, train_ids, n_train);
            upload_codebooks(x);
            if (!n_local) raise(SUCO_ERR_CONFIG, "shard owns no points (n too small for this block size)");
            finalize_shard(x);
        } catch (...) {
            delete x;
            throw;
        }
        *out = x;
    });
}

int suco_gpu_shard_info(const suco_gpu_index* x, uint64_t* n_global, uint64_t* n_local, uint32_t* block,
                        uint32_t* shard, uint32_t* num_shards) {
    return guarded([&] {
        if (!x) raise(SUCO_ERR_CONTRACT, "index is null");
        if (n_global) *n_global = x->n_global;
        if (n_local) *n_local = x->host.n;
        if (block) *block = x->block;
        if (shard) *shard = x->shard;
        if (num_shards) *num_shards = x->num_shards;
    });
}

int suco_gpu_shard_knn_query_batch_device(const suco_gpu_index* x, suco_comm* comm, const float* d_queries,
                                          uint64_t nq, uint32_t qlen, const suco_collision_params* p, uint32_t* d_ids,
                                          double* d_dists, void* stream, suco_gpu_query_ctx* ctx) {
    return guarded([&] {
        check_shard_query(x, comm, qlen, p);
        check_ctx(x, ctx);
        if (nq == 0) return;
        if (!d_queries || !d_ids || !d_dists) raise(SUCO_ERR_CONTRACT, "null buffer");
        DeviceGuard g(x->device);
        CtxLease lease(x, ctx);
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : lease.c->own;
        shard_run(x, lease.c, comm, nullptr, d_queries, nq, qlen, p, d_ids, d_dists, nullptr, nullptr, st);
    });
}

int suco_gpu_shard_knn_query_batch(const suco_gpu_index* x, suco_comm* comm, const float* queries, uint64_t nq,
                                   uint32_t qlen, const suco_collision_params* p, uint32_t* ids, double* dists,
                                   suco_gpu_query_ctx* ctx) {
    return guarded([&] {
        check_shard_query(x, comm, qlen, p);
        check_ctx(x, ctx);
        if (nq == 0) return;
        if (!queries || !ids || !dists) raise(SUCO_ERR_CONTRACT, "null buffer");
        DeviceGuard g(x->device);
        CtxLease lease(x, ctx);
        shard_run(x, lease.c, comm, queries, nullptr, nq, qlen, p, nullptr, nullptr, ids, dists, lease.c->own);
        CUDA_TRY(cudaStreamSynchronize(lease.c->own));
    });
}

}  // extern "C"
