// C-ABI, stand-alone entry points: exact kNN and SC-Linear over an index's
// device rows, and each query/build stage's kernel on
// host inputs (parity tests of the reference's free functions).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "build.h"
#include "capi_internal.h"

using namespace suco_gpu;

namespace {

// SC-Linear (sc_linear.cpp:49-121) over the index's device rows and layout.
struct ScScratch {
    DevBuf<uint32_t> sub_off;
    DevBuf<uint8_t> consec, scratch;
    DevBuf<float> q;
    ScArgs a{};
};

void sc_setup(const suco_gpu_index* x, ScScratch& w, uint32_t B, uint64_t m, cudaStream_t st) {
    const HostLayout& L = x->host.layout;
    const uint64_t n = x->host.n;
    std::vector<uint32_t> off(L.ns + 1, 0);
    std::vector<uint8_t> consec(L.ns, 0);
    for (uint32_t s = 0; s < L.ns; ++s) {
        off[s + 1] = off[s] + L.sizes[s];
        bool run = L.sizes[s] > 0;  // consecutive_start (subspace.cpp:93-102)
        for (uint32_t j = off[s] + 1; j < off[s + 1]; ++j) run = run && L.dims[j] == L.dims[j - 1] + 1;
        consec[s] = run;
    }
    w.sub_off.reserve(L.ns + 1);
    w.consec.reserve(L.ns);
    CUDA_TRY(cudaMemcpyAsync(w.sub_off.p, off.data(), off.size() * 4, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(w.consec.p, consec.data(), consec.size(), cudaMemcpyHostToDevice, st));
    w.q.reserve(uint64_t(B) * x->host.d);
    w.scratch.reserve(sc_batch_bytes(n, B, m));
    w.a.data = x->data.p;
    w.a.n = n;
    w.a.d = x->host.d;
    w.a.ns = L.ns;
    w.a.dims = x->dims.p;
    w.a.sub_off = w.sub_off.p;
    w.a.consec = w.consec.p;
    w.a.q = w.q.p;
    w.a.scratch = w.scratch.p;
}

// queries per SC-Linear batch: the n distance keys (+ scores) of each within about 2 GB
uint32_t sc_batch_size(uint64_t n, uint64_t nq) {
    const uint64_t per = n * 9 + 64;
    return static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(nq, (2ull << 30) / per)));
}

void check_sc_query(const suco_gpu_index* x, uint32_t qlen) {
    if (!x) raise(SUCO_ERR_CONTRACT, "index is null");
    if (x->num_shards > 1) raise(SUCO_ERR_CONTRACT, "SC-Linear needs the full index");
    check_query_len(qlen, x->host.d);  // sc_linear.cpp:55-58
}

}  // namespace

extern "C" {

// exact_knn (eval.hpp:29, eval.cpp:28-62) for a batch: the re-rank kernels over every id.
int suco_gpu_exact_knn_batch(const suco_gpu_index* x, const float* queries, uint64_t nq, uint32_t qlen, uint32_t k,
                             uint32_t* ids, double* dists) {
    return guarded([&] {
        if (!x) raise(SUCO_ERR_CONTRACT, "index is null");
        if (x->num_shards > 1) raise(SUCO_ERR_CONTRACT, "exact kNN needs the full index");
        const uint64_t n = x->host.n;
        check_query_len(qlen, x->host.d);
        if (k < 1 || k > n) {
            raise(SUCO_ERR_CONTRACT, "k must be in [1, n]; got k = " + std::to_string(k) + ", n = " + std::to_string(n));
        }
        if (nq == 0) return;
        if (!queries || !ids || !dists) raise(SUCO_ERR_CONTRACT, "null buffer");
        DeviceGuard g(x->device);
        OwnStream os;
        cudaStream_t st = os.s;
        // tiles of queries (k > 32: one query per launch, its n scored rows in scratch)
        const uint64_t tile = k > 32 ? 1 : std::min<uint64_t>(nq, 8192);
        DevBuf<float> dq;
        DevBuf<uint32_t> di;
        DevBuf<double> dd, all_d;
        DevBuf<uint32_t> all_id;
        dq.reserve(tile * qlen);
        di.reserve(tile * k);
        dd.reserve(tile * k);
        if (k > 32) {
            all_d.reserve(n);
            all_id.reserve(n);
        }
        for (uint64_t q0 = 0; q0 < nq; q0 += tile) {
            const uint64_t nt = std::min<uint64_t>(tile, nq - q0);
            CUDA_TRY(cudaMemcpyAsync(dq.p, queries + q0 * qlen, nt * qlen * 4, cudaMemcpyHostToDevice, st));
            RerankArgs ra{};
            rerank_args(x, ra);
            ra.queries = dq.p;
            ra.cands = nullptr;
            ra.identity = true;
            ra.m = n;
            ra.k = k;
            ra.out_ids = di.p;
            ra.out_dists = dd.p;
            ra.all_d = all_d.p;
            ra.all_id = all_id.p;
            CUDA_TRY(launch_rerank(ra, nt, st));
            CUDA_TRY(cudaMemcpyAsync(ids + q0 * k, di.p, nt * k * 4, cudaMemcpyDeviceToHost, st));
            CUDA_TRY(cudaMemcpyAsync(dists + q0 * k, dd.p, nt * k * 8, cudaMemcpyDeviceToHost, st));
        }
        CUDA_TRY(cudaStreamSynchronize(st));
    });
}

int suco_gpu_sc_scores(const suco_gpu_index* x, const float* query, uint32_t qlen, double alpha, uint32_t* scores) {
    return guarded([&] {
        check_sc_query(x, qlen);
        // the reference leaves alpha unchecked here (c > n would index past the order array)
        if (!(alpha > 0.0) || alpha > 1.0) raise(SUCO_ERR_CONFIG, "alpha must be in (0, 1], got " + std::to_string(alpha));
        if (!query || !scores) raise(SUCO_ERR_CONTRACT, "null buffer");
        DeviceGuard g(x->device);
        OwnStream os;
        cudaStream_t st = os.s;
        const uint64_t n = x->host.n;
        ScScratch w;
        sc_setup(x, w, 1, 1, st);
        DevBuf<uint8_t> sc;
        sc.reserve(n);
        const uint64_t c = std::min<uint64_t>(suco_collision_count(alpha, n), n);
        CUDA_TRY(cudaMemcpyAsync(w.q.p, query, qlen * 4, cudaMemcpyHostToDevice, st));
        CUDA_TRY(launch_sc_batch(w.a, 1, c, 1, nullptr, sc.p, st));
        std::vector<uint8_t> h(n);
        CUDA_TRY(cudaMemcpyAsync(h.data(), sc.p, n, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        for (uint64_t i = 0; i < n; ++i) scores[i] = h[i];
    });
}

int suco_gpu_sc_linear_batch(const suco_gpu_index* x, const float* queries, uint64_t nq, uint32_t qlen,
                             const suco_collision_params* p, uint32_t* ids, double* dists) {
    return guarded([&] {
        if (!x) raise(SUCO_ERR_CONTRACT, "index is null");
        validate_params(p, x->host.n);  // sc_linear.cpp:97, before the query-length check
        check_sc_query(x, qlen);
        if (nq == 0) return;
        if (!queries || !ids || !dists) raise(SUCO_ERR_CONTRACT, "null buffer");
        DeviceGuard g(x->device);
        OwnStream os;
        cudaStream_t st = os.s;
        const uint64_t n = x->host.n;
        const uint64_t c = std::min<uint64_t>(suco_collision_count(p->alpha, n), n);
        const uint64_t m = std::min<uint64_t>(suco_candidate_count(p->beta, n, p->k), n);
        const uint32_t B = x->tune.sc_batch ? static_cast<uint32_t>(std::min<uint64_t>(x->tune.sc_batch, nq))
                                            : sc_batch_size(n, nq);
        ScScratch w;
        sc_setup(x, w, B, m, st);
        DevBuf<uint32_t> cands, di, all_id;
        DevBuf<double> dd, all_d;
        cands.reserve(uint64_t(B) * m);
        di.reserve(uint64_t(B) * p->k);
        dd.reserve(uint64_t(B) * p->k);
        if (p->k > 32) {
            all_d.reserve(uint64_t(B) * m);
            all_id.reserve(uint64_t(B) * m);
        }
        for (uint64_t q0 = 0; q0 < nq; q0 += B) {
            const uint32_t nb = static_cast<uint32_t>(std::min<uint64_t>(B, nq - q0));
            CUDA_TRY(cudaMemcpyAsync(w.q.p, queries + q0 * qlen, uint64_t(nb) * qlen * 4, cudaMemcpyHostToDevice, st));
            CUDA_TRY(launch_sc_batch(w.a, nb, c, m, cands.p, nullptr, st));
            RerankArgs ra{};
            rerank_args(x, ra);
            ra.queries = w.q.p;
            ra.cands = cands.p;
            ra.m = m;
            ra.k = p->k;
            ra.out_ids = di.p;
            ra.out_dists = dd.p;
            ra.all_d = all_d.p;
            ra.all_id = all_id.p;
            CUDA_TRY(launch_rerank(ra, nb, st));
            CUDA_TRY(cudaMemcpyAsync(ids + q0 * p->k, di.p, uint64_t(nb) * p->k * 4, cudaMemcpyDeviceToHost, st));
            CUDA_TRY(cudaMemcpyAsync(dists + q0 * p->k, dd.p, uint64_t(nb) * p->k * 8, cudaMemcpyDeviceToHost, st));
        }
        CUDA_TRY(cudaStreamSynchronize(st));
    });
}

int suco_gpu_centroid_distances(const float* half_query, uint32_t dim, const float* centroids, uint32_t k_half,
                                double* dists, uint32_t* order) {
    return guarded([&] {
        if (k_half < 1) raise(SUCO_ERR_CONTRACT, "k_half must be >= 1");   // query.cpp:44-49
        if (dim == 0) raise(SUCO_ERR_CONTRACT, "query half is empty");
        DeviceGuard g(0);
        DevBuf<float> q, c;
        DevBuf<double> dd;
        DevBuf<uint32_t> oo;
        q.reserve(dim);
        c.reserve(uint64_t(k_half) * dim);
        dd.reserve(k_half);
        oo.reserve(k_half);
        CUDA_TRY(cudaMemcpy(q.p, half_query, dim * 4, cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(c.p, centroids, uint64_t(k_half) * dim * 4, cudaMemcpyHostToDevice));
        CUDA_TRY(launch_centroid_distances(q.p, dim, c.p, k_half, dd.p, oo.p, 0));
        CUDA_TRY(cudaMemcpy(dists, dd.p, k_half * 8, cudaMemcpyDeviceToHost));
        CUDA_TRY(cudaMemcpy(order, oo.p, k_half * 4, cudaMemcpyDeviceToHost));
    });
}

int suco_gpu_dynamic_activation(double alpha, uint64_t n, const double* d1, const uint32_t* o1, const double* d2,
                                const uint32_t* o2, uint32_t k_half, const uint64_t* offsets, uint32_t* c1, uint32_t* c2,
                                uint64_t* cumulative, double* sum_dist, uint64_t cap, uint64_t* count) {
    return guarded([&] {
        // check_traversal_args, query.cpp:16-30
        if (!(alpha > 0.0) || alpha > 1.0) raise(SUCO_ERR_CONTRACT, "alpha must be in (0, 1]");
        if (k_half < 1) raise(SUCO_ERR_CONTRACT, "imi has no cells");
        const uint64_t K = uint64_t(k_half) * k_half;
        if (offsets[K] != n) {
            raise(SUCO_ERR_CONTRACT, "imi holds " + std::to_string(offsets[K]) + " ids but n = " + std::to_string(n));
        }
        if (n > 0xFFFFFFFFull) raise(SUCO_ERR_CONTRACT, "n exceeds 32-bit point-id capacity");
        DeviceGuard g(0);
        std::vector<uint32_t> sizes(K);
        for (uint64_t c = 0; c < K; ++c) sizes[c] = static_cast<uint32_t>(offsets[c + 1] - offsets[c]);
        DevBuf<double> dd1, dd2, sums;
        DevBuf<uint32_t> oo1, oo2, sz, cells, nc;
        DevBuf<uint64_t> cum;
        dd1.reserve(k_half), dd2.reserve(k_half), oo1.reserve(k_half), oo2.reserve(k_half);
        sz.reserve(K), cells.reserve(K), sums.reserve(K), cum.reserve(K), nc.reserve(1);
        CUDA_TRY(cudaMemcpy(dd1.p, d1, k_half * 8, cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(dd2.p, d2, k_half * 8, cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(oo1.p, o1, k_half * 4, cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(oo2.p, o2, k_half * 4, cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(sz.p, sizes.data(), K * 4, cudaMemcpyHostToDevice));
        CUDA_TRY(launch_da_only(dd1.p, oo1.p, dd2.p, oo2.p, k_half, sz.p, suco_collision_count(alpha, n), cells.p, nc.p,
                                sums.p, cum.p, 0));
        uint32_t got = 0;
        CUDA_TRY(cudaMemcpy(&got, nc.p, 4, cudaMemcpyDeviceToHost));
        *count = got;
        const uint64_t w = std::min<uint64_t>(got, cap);
        std::vector<uint32_t> cl(w);
        if (w) {
            CUDA_TRY(cudaMemcpy(cl.data(), cells.p, w * 4, cudaMemcpyDeviceToHost));
            CUDA_TRY(cudaMemcpy(sum_dist, sums.p, w * 8, cudaMemcpyDeviceToHost));
            CUDA_TRY(cudaMemcpy(cumulative, cum.p, w * 8, cudaMemcpyDeviceToHost));
        }
        for (uint64_t i = 0; i < w; ++i) {
            c1[i] = cl[i] / k_half;
            c2[i] = cl[i] % k_half;
        }
        if (got > cap) raise(SUCO_ERR_CONTRACT, "cell output capacity too small");
    });
}

int suco_gpu_rerank(const float* data, uint64_t n, uint32_t d, const float* query, uint32_t qlen,
                    const uint32_t* candidates, uint64_t m, uint32_t k, uint32_t* ids, double* dists) {
    return guarded([&] {
        // query.cpp:159-176
        if (qlen != d) {
            raise(SUCO_ERR_CONTRACT, "query length " + std::to_string(qlen) + " does not match dataset d = " +
                                         std::to_string(d));
        }
        if (k < 1) raise(SUCO_ERR_CONTRACT, "k must be >= 1");
        if (m < k) raise(SUCO_ERR_CONTRACT, "k = " + std::to_string(k) + " exceeds the " + std::to_string(m) + " candidates");
        for (uint64_t i = 0; i < m; ++i) {
            if (candidates[i] >= n) raise(SUCO_ERR_CONTRACT, "candidate id " + std::to_string(candidates[i]) + " out of range");
        }
        DeviceGuard g(0);
        const Tuning tune = tuning_from_env();
        DevBuf<float> dd, qq;
        DevBuf<uint32_t> cc, oi, ai;
        DevBuf<double> od, ad;
        dd.reserve(n * d), qq.reserve(d), cc.reserve(m), oi.reserve(k), od.reserve(k);
        CUDA_TRY(cudaMemcpy(dd.p, data, n * d * 4, cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(qq.p, query, d * 4, cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(cc.p, candidates, m * 4, cudaMemcpyHostToDevice));
        RerankArgs ra{};
        ra.data = dd.p;
        ra.n = n;
        ra.d = d;
        ra.queries = qq.p;
        ra.cands = cc.p;
        ra.m = m;
        ra.k = k;
        ra.out_ids = oi.p;
        ra.out_dists = od.p;
        ra.u8_regs = tune.rerank_u8_regs;
        ra.pipe = tune.rerank_pipe == 2 ? 0 : tune.rerank_pipe == 1 ? 1 : 2;
        DevBuf<uint8_t> d8;
        {
            DevBuf<unsigned int> st;
            st.reserve(3);
            unsigned int h[3] = {0, 0, 0};
            CUDA_TRY(cudaMemset(st.p, 0, 12));
            CUDA_TRY(launch_int_stats(dd.p, n * d, st.p, 0));
            CUDA_TRY(cudaMemcpy(h, st.p, 12, cudaMemcpyDeviceToHost));
            float mx;
            std::memcpy(&mx, &h[1], 4);
            ra.data_int_max = (h[0] == 0 && mx <= 1048576.f) ? mx : -1.f;
            if (h[0] == 0 && h[2] == 0 && mx <= 255.f && d <= 512 && !tune.no_u8) {
                ra.dpad = (d + 15) / 16 * 16;
                d8.reserve(n * ra.dpad);
                CUDA_TRY(launch_pack_u8(dd.p, n, d, ra.dpad, d8.p, 0));
                ra.data8 = d8.p;
            }
        }
        if (k > 32) {
            ad.reserve(m), ai.reserve(m);
            ra.all_d = ad.p;
            ra.all_id = ai.p;
        }
        CUDA_TRY(launch_rerank(ra, 1, 0));
        CUDA_TRY(cudaMemcpy(ids, oi.p, k * 4, cudaMemcpyDeviceToHost));
        CUDA_TRY(cudaMemcpy(dists, od.p, k * 8, cudaMemcpyDeviceToHost));
    });
}

int suco_gpu_kmeans(const float* points, uint64_t n, uint32_t dim, uint32_t k, uint32_t iterations, uint64_t seed,
                    int device, float* centroids, uint32_t* assignments, uint32_t* repaired, uint32_t* num_repaired) {
    return guarded([&] {
        // kmeans.cpp:121-126
        if (k < 1) raise(SUCO_ERR_CONFIG, "kmeans: k must be >= 1");
        if (iterations < 1) raise(SUCO_ERR_CONFIG, "kmeans: iterations must be >= 1");
        if (n < k) raise(SUCO_ERR_CONFIG, "kmeans: n = " + std::to_string(n) + " is smaller than k = " + std::to_string(k));
        if (n > 0xFFFFFFFFull) raise(SUCO_ERR_CONTRACT, "kmeans: n exceeds 32-bit point-id capacity");
        DeviceGuard g(device);
        kmeans_device_host_io(points, n, dim, k, iterations, seed, centroids, assignments, repaired, num_repaired);
    });
}

int suco_gpu_build_imi(const uint32_t* first, const uint32_t* second, uint64_t n, uint32_t k_half, uint64_t* offsets,
                       uint32_t* ids) {
    return guarded([&] {
        if (k_half < 1) raise(SUCO_ERR_CONTRACT, "build_imi: k_half must be >= 1");  // index.cpp:72-76
        if (n > 0xFFFFFFFFull) raise(SUCO_ERR_CONTRACT, "build_imi: n exceeds 32-bit point-id capacity");
        for (uint64_t i = 0; i < n; ++i) {
            if (first[i] >= k_half || second[i] >= k_half) {
                raise(SUCO_ERR_CONTRACT, "assignment out of range at point " + std::to_string(i));
            }
        }
        DeviceGuard g(0);
        build_imi_host_io(first, second, n, k_half, offsets, ids);
    });
}

}  // extern "C"
