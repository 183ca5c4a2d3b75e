// C-ABI implementation (include/suco_b200.h), core: validation in the
// reference's order, index upload/build, query contexts, and the query
// pipeline
//   traverse (thread / warp per query x subspace) -> select (dense bit-sliced
//   blocks or clusters per query) -> rerank (CTA per query)
// on a context's three streams, tiled over the query batch so the per-query
// scratch (retrieved cells, candidates) stays within the memory budget.
// Shards: capi_shard.cu; stand-alone stages: capi_stage.cu; vecs I/O: capi_io.cu.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "build.h"
#include "capi_internal.h"

using namespace suco_gpu;

namespace suco_gpu {

thread_local std::string g_err;

DeviceGuard::DeviceGuard(int dev) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        raise(SUCO_ERR_INTERNAL, "no CUDA device available: the SuCo B200 path has no CPU fallback");
    }
    if (dev < 0 || dev >= count) raise(SUCO_ERR_INTERNAL, "CUDA device " + std::to_string(dev) + " does not exist");
    CUDA_TRY(cudaGetDevice(&prev));
    if (prev != dev) CUDA_TRY(cudaSetDevice(dev));
}

OwnStream::OwnStream() { CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }

void check_query_len(uint32_t qlen, uint32_t d) {  // query.cpp:203-206
    if (qlen != d) {
        raise(SUCO_ERR_CONTRACT, "query length " + std::to_string(qlen) + " does not match dataset d = " +
                                     std::to_string(d));
    }
}

}  // namespace suco_gpu

void suco_gpu_query_ctx::Slot::release_all() {
    q.release(), cells.release(), ncells.release(), cands.release(), out_ids.release(), all_id.release();
    dhist.release(), dT.release(), dquota.release(), dbase.release(), dsample.release(), dcbuf.release();
    dccnt.release(), dL.release(), dflag.release(), dh2.release(), out_d.release(), all_d.release();
}

suco_gpu_query_ctx::~suco_gpu_query_ctx() {
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    for (cudaStream_t t : pipe) {
        if (t) cudaStreamSynchronize(t);
    }
    if (own) cudaStreamSynchronize(own);
    for (cudaEvent_t e : events) cudaEventDestroy(e);
    for (Slot& sl : slot) {
        for (cudaEvent_t e : {sl.trav, sl.sel, sl.rr, sl.selmain}) {
            if (e) cudaEventDestroy(e);
        }
        sl.release_all();
    }
    for (cudaEvent_t e : {ev_in, ev_out}) {
        if (e) cudaEventDestroy(e);
    }
    sh_tot.release(), sh_tot_all.release(), sh_ties.release(), sh_ties_all.release(), sh_qblk.release();
    sh_counts.release(), sh_ids.release(), sh_ids_all.release(), sh_need.release(), sh_sq.release(), sh_sq_all.release();
    sh_s17.release(), sh_gt.release(), sh_gts.release(), sh_nflag.release();
    stat_cum.release();
    for (cudaStream_t t : pipe) {
        if (t) cudaStreamDestroy(t);
    }
    if (own) cudaStreamDestroy(own);
    if (prev >= 0) cudaSetDevice(prev);
}

suco_gpu_index::~suco_gpu_index() {
    for (suco_gpu_query_ctx* c : pool) delete c;  // sets its own device
    if (own) cudaStreamDestroy(own);
}

namespace suco_gpu {

// ------------------------------------------------------------ query contexts
suco_gpu_query_ctx* ctx_new(const suco_gpu_index* x) {
    auto* c = new suco_gpu_query_ctx();
    c->index = x;
    c->device = x->device;
    try {
        CUDA_TRY(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking));
        int least = 0, greatest = 0;
        CUDA_TRY(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        // traverse and rerank (short, many small CTAs) get priority so they fill the SMs that
        // select's long CTAs leave idle; the dense select's fallback (a few query blocks,
        // latency-bound) runs beside the re-rank of the unflagged queries, its CTAs first
        CUDA_TRY(cudaStreamCreateWithPriority(&c->pipe[0], cudaStreamNonBlocking, greatest));
        CUDA_TRY(cudaStreamCreateWithPriority(&c->pipe[1], cudaStreamNonBlocking, least));
        const int rr_prio = greatest < least ? greatest + 1 : greatest;
        CUDA_TRY(cudaStreamCreateWithPriority(&c->pipe[2], cudaStreamNonBlocking, rr_prio));
        CUDA_TRY(cudaStreamCreateWithPriority(&c->pipe[3], cudaStreamNonBlocking, greatest));
        for (auto& sl : c->slot) {
            for (cudaEvent_t* e : {&sl.trav, &sl.sel, &sl.rr, &sl.selmain}) {
                CUDA_TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
            }
        }
        CUDA_TRY(cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&c->ev_out, cudaEventDisableTiming));
        for (cudaStream_t t : {c->own, c->pipe[0], c->pipe[1], c->pipe[2], c->pipe[3]}) apply_l2_window(x, t);
    } catch (...) {
        delete c;
        throw;
    }
    return c;
}

CtxLease::CtxLease(const suco_gpu_index* xi, suco_gpu_query_ctx* given) : x(xi), c(given), pooled(given == nullptr) {
    if (given) {
        check_ctx(x, given);
        return;
    }
    {
        std::lock_guard<std::mutex> lk(x->pool_mu);
        if (!x->pool.empty()) {
            c = x->pool.back();
            x->pool.pop_back();
        }
    }
    if (!c) c = ctx_new(x);
    c->profile = false;
}

CtxLease::~CtxLease() {
    if (!pooled || !c) return;
    std::lock_guard<std::mutex> lk(x->pool_mu);
    x->pool.push_back(c);
}

void check_ctx(const suco_gpu_index* x, const suco_gpu_query_ctx* c) {
    if (c && c->index != x) raise(SUCO_ERR_CONTRACT, "query context belongs to another index");
}

// ------------------------------------------------------------ device upload
void create_index_stream(suco_gpu_index* x) { CUDA_TRY(cudaStreamCreateWithFlags(&x->own, cudaStreamNonBlocking)); }

}  // namespace suco_gpu

namespace {

void check_dataset(const float* data, uint64_t n, uint32_t d) {
    if (n < 1 || d < 1) raise(SUCO_ERR_CONTRACT, "dataset requires n >= 1 and d >= 1");
    if (!data) raise(SUCO_ERR_CONTRACT, "dataset buffer is null");
}

// Dataset finiteness (core.cpp:15-19), checked on the device after upload.
void check_finite_device(const float* d_data, uint64_t count, cudaStream_t st) {
    DevBuf<unsigned long long> flag;
    flag.reserve(1);
    const unsigned long long init = ~0ull;
    unsigned long long got = 0;
    CUDA_TRY(cudaMemcpyAsync(flag.p, &init, sizeof init, cudaMemcpyHostToDevice, st));
    CUDA_TRY(launch_check_finite(d_data, count, reinterpret_cast<int*>(flag.p), st));
    CUDA_TRY(cudaMemcpyAsync(&got, flag.p, sizeof got, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (got != ~0ull) raise(SUCO_ERR_CONTRACT, "dataset component " + std::to_string(got) + " is not finite");
}

}  // namespace

namespace suco_gpu {

// Copies `bytes` of pageable host memory to the device through four pinned 64 MB stages: host
// threads fill a stage (memcpy split eight ways) while the DMA engine drains the previous ones.
// A single cudaMemcpy from pageable memory ran at about 10 GB/s (the driver's own staging);
// device or pinned sources take one cudaMemcpyAsync.
void copy_rows_to_device(void* dst, const void* src, uint64_t bytes, cudaStream_t st) {
    cudaPointerAttributes pa{};
    const bool pageable = cudaPointerGetAttributes(&pa, src) == cudaSuccess && pa.type == cudaMemoryTypeUnregistered;
    cudaGetLastError();  // (clears the error some drivers report for unregistered pointers)
    constexpr uint64_t kStage = 64ull << 20;
    constexpr int kStages = 4, kThreads = 8;
    if (!pageable || bytes < 4 * kStage) {
        CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st));
        return;
    }
    unsigned char* stage[kStages] = {};
    cudaEvent_t done[kStages] = {};
    struct Cleanup {
        unsigned char** s;
        cudaEvent_t* e;
        ~Cleanup() {
            for (int i = 0; i < kStages; ++i) {
                if (e[i]) cudaEventSynchronize(e[i]), cudaEventDestroy(e[i]);
                if (s[i]) cudaFreeHost(s[i]);
            }
        }
    } cleanup{stage, done};
    for (int i = 0; i < kStages; ++i) {
        CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&stage[i]), kStage, cudaHostAllocDefault));
        CUDA_TRY(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
    }
    const unsigned char* in = static_cast<const unsigned char*>(src);
    unsigned char* out = static_cast<unsigned char*>(dst);
    uint64_t chunk = 0;
    for (uint64_t off = 0; off < bytes; off += kStage, ++chunk) {
        const int b = static_cast<int>(chunk % kStages);
        const uint64_t len = std::min<uint64_t>(kStage, bytes - off);
        if (chunk >= kStages) CUDA_TRY(cudaEventSynchronize(done[b]));  // the stage's previous DMA
        std::thread th[kThreads];
        const uint64_t part = (len + kThreads - 1) / kThreads;
        for (int t = 0; t < kThreads; ++t) {
            const uint64_t lo = std::min<uint64_t>(len, t * part), hi = std::min<uint64_t>(len, lo + part);
            th[t] = std::thread([=] { if (hi > lo) std::memcpy(stage[b] + lo, in + off + lo, hi - lo); });
        }
        for (auto& t : th) t.join();
        CUDA_TRY(cudaMemcpyAsync(out + off, stage[b], len, cudaMemcpyHostToDevice, st));
        CUDA_TRY(cudaEventRecord(done[b], st));
    }
}

// data == nullptr: the rows are already in x->data (streamed from a vecs file).
void upload_data(suco_gpu_index* x, const float* data, uint64_t n, uint32_t d) {
    if (data) {
        x->data.reserve(n * d);
        // host or device memory (UVA): rows already on the GPU are copied device to device
        copy_rows_to_device(x->data.p, data, n * d * sizeof(float), x->own);
    }
    check_finite_device(x->data.p, n * d, x->own);
    // integer certificate (values integral, |v| <= 2^20) for the exact fp32 rerank chains
    DevBuf<unsigned int> st;
    st.reserve(3);
    unsigned int h[3] = {0, 0, 0};
    CUDA_TRY(cudaMemsetAsync(st.p, 0, 12, x->own));
    CUDA_TRY(launch_int_stats(x->data.p, n * d, st.p, x->own));
    CUDA_TRY(cudaMemcpyAsync(h, st.p, 12, cudaMemcpyDeviceToHost, x->own));
    CUDA_TRY(cudaStreamSynchronize(x->own));
    float mx;
    std::memcpy(&mx, &h[1], 4);
    x->data_int_max = (h[0] == 0 && mx <= 1048576.f) ? mx : -1.f;
    // u8-valued rows (integers in [0, 255]): a byte copy for the exact integer re-rank, whose
    // squared distances (< 2^32) are the reference's fp64 values in any summation order
    x->dpad = 0;
    if (h[0] == 0 && h[2] == 0 && mx <= 255.f && d <= 512 && !x->tune.no_u8) {
        x->dpad = (d + 15) / 16 * 16;
        x->data8.reserve(n * x->dpad);
        CUDA_TRY(launch_pack_u8(x->data.p, n, d, x->dpad, x->data8.p, x->own));
    }
    // other rows: an int8 copy with per-row bound terms for the re-rank's certified screen (a
    // quarter of the f32 row bytes; rerank_q8_kernel)
    x->qpad = x->qrec = 0;
    // (d <= 128: rerank_q8p / rerank_q8 kernels; 128 < d <= 1024: rerank_q8w, prefix records only)
    if (!x->dpad && x->tune.q8 && d % 4 == 0 && (d <= 128 || (d <= 1024 && x->tune.q8_prefix == 3))) {
        x->qpad = (d + 15) / 16 * 16;
        // Past the prefix: the prefix-bound layout (meta0 and the prefix dims in the first qsplit
        // bytes, the rest and meta1 after them: pack_q8_kernel); whole 64-byte granules per record
        const uint32_t nw = x->qpad / 16, pre = x->tune.q8_prefix;
        x->qpre = nw > pre ? pre : 0u;
        x->qsplit = x->qpre ? (16 + 16 * x->qpre + 31) / 32 * 32 : 0u;
        x->qrec = x->qpre ? (x->qsplit + (nw - x->qpre + 1) * 16 + 63) / 64 * 64 : (x->qpad + 16 + 63) / 64 * 64;
        x->q8.reserve(n * x->qrec);
        x->q8_rows = n;
        CUDA_TRY(launch_pack_q8(x->data.p, n, d, x->qpad, x->qrec, x->qpre, x->qsplit, x->q8.p, x->own));
        CUDA_TRY(cudaStreamSynchronize(x->own));
    }
}

// Layout + centroid tables on the device, from x->host.
void upload_codebooks(suco_gpu_index* x) {
    const HostIndex& h = x->host;
    const uint32_t ns = h.layout.ns;
    std::vector<SubDesc> sd(ns);
    std::vector<float> cent;
    uint32_t pos = 0;
    x->hmax = 0;
    for (uint32_t s = 0; s < ns; ++s) {
        SubDesc& d = sd[s];
        d.h1 = h.layout.h1(s);
        d.h2 = h.layout.h2(s);
        d.dims1 = pos;
        d.dims2 = pos + d.h1;
        pos += h.layout.sizes[s];
        d.cent1 = cent.size();
        cent.insert(cent.end(), h.cent1[s].begin(), h.cent1[s].end());
        d.cent2 = cent.size();
        cent.insert(cent.end(), h.cent2[s].begin(), h.cent2[s].end());
        x->hmax = std::max({x->hmax, d.h1, d.h2});
    }
    x->dims.reserve(h.layout.dims.size());
    CUDA_TRY(cudaMemcpyAsync(x->dims.p, h.layout.dims.data(), h.layout.dims.size() * 4, cudaMemcpyHostToDevice, x->own));
    x->sub.reserve(ns);
    CUDA_TRY(cudaMemcpyAsync(x->sub.p, sd.data(), ns * sizeof(SubDesc), cudaMemcpyHostToDevice, x->own));
    x->cent.reserve(cent.size());
    CUDA_TRY(cudaMemcpyAsync(x->cent.p, cent.data(), cent.size() * 4, cudaMemcpyHostToDevice, x->own));
    CUDA_TRY(cudaStreamSynchronize(x->own));
}

// Keep the IMI ids (+ slab offsets) L2-resident across the query stream: the cluster select's
// id loads are L2-latency bound, and the candidate writes and re-rank row gathers would otherwise
// evict them (measured: 93 % L2 hits, i.e. nearly every 256-load wave waited on a DRAM miss).
// The persisting carve-out is a device setting (at index creation); the window goes on every
// query context's streams.
void set_l2_persisting(const suco_gpu_index* x) {
    int max_persist = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, x->device));
    if (max_persist <= 0) return;
    const size_t want = x->ids.cap * sizeof(uint32_t);
    CUDA_TRY(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min<size_t>(want, static_cast<size_t>(max_persist))));
}

void apply_l2_window(const suco_gpu_index* x, cudaStream_t st) {
    int max_persist = 0, max_window = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, x->device));
    CUDA_TRY(cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, x->device));
    if (max_persist <= 0 || max_window <= 0 || !x->ids.p) return;
    const size_t want = x->ids.cap * sizeof(uint32_t);
    const size_t persist = std::min<size_t>(want, static_cast<size_t>(max_persist));
    cudaStreamAttrValue v{};
    v.accessPolicyWindow.base_ptr = x->ids.p;
    v.accessPolicyWindow.num_bytes = std::min<size_t>(want, static_cast<size_t>(max_window));
    v.accessPolicyWindow.hitRatio =
        std::min(1.0f, static_cast<float>(persist) / static_cast<float>(v.accessPolicyWindow.num_bytes));
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    CUDA_TRY(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v));
}

// The select stage's tables: dense point codes (N_s <= 16 and the masks fit), the half-width
// mode for large N_s * K (config 5), else the cluster-counting select's slab offsets.
void finalize_dense(suco_gpu_index* x, bool allow_half) {
    const uint32_t ns = x->host.layout.ns;
    const uint64_t n = x->host.n;
    const Tuning& t = x->tune;
    x->dense = (dense_supported(ns, x->K) || dense_wide_supported(ns, x->K)) && t.dense;
    // tables past 32-bit masks in shared memory (config 5: 8 x 10,000 cells) take the half-width
    // mode; SUCO_DENSE_HALF=0 keeps them on the cluster-counting select (2 forces it: tests)
    x->dense_half = allow_half && (!x->dense || t.dense_half == 2) && t.dense && t.dense_half != 0 &&
                    dense_half_supported(ns, x->K);
    if (x->dense_half) {
        x->dense = true;
        // whole last piece of any single-pass piece size, plus two 64-point tiles (the fused pass
        // loads the codes two tiles ahead of the one it scores)
        const uint64_t n_pad = (n + kMaxPiece - 1) / kMaxPiece * kMaxPiece + 128;
        x->codes.reserve(n_pad * 8);
        x->dense_hgroup = ns == 8 && !t.dense_pair;
        CUDA_TRY(launch_dense_codes_half(x->ids.p, x->cell_off.p, n, n_pad, ns, x->K, x->codes.p,
                                         x->dense_hgroup ? 1u : 0u, t.dense_sched, x->own));
    } else if (x->dense) {
        x->codes.reserve((n + kDenseCodePad) * (ns > 8 ? 16 : 8));
        CUDA_TRY(launch_dense_codes(x->ids.p, x->cell_off.p, n, ns, x->K, x->codes.p, t.dense_sched, x->own));
    }
    if (!x->dense) {
        x->sel = plan_select(n, ns, t.cluster);
        x->slab_off.reserve(uint64_t(ns) * x->K * (x->sel.nslabs + 1));
        CUDA_TRY(launch_slab_offsets(x->cell_off.p, x->ids.p, n, ns, x->K, x->sel.CH, x->sel.nslabs, x->slab_off.p,
                                     x->own));
    }
    CUDA_TRY(cudaStreamSynchronize(x->own));
}

}  // namespace suco_gpu

namespace {

// Cell sizes, select tables and the L2 carve-out from the device-resident CSR.
void finalize_device(suco_gpu_index* x) {
    const uint32_t ns = x->host.layout.ns;
    x->K = x->host.p.k_half * x->host.p.k_half;
    x->cell_size.reserve(uint64_t(ns) * x->K);
    CUDA_TRY(launch_cell_sizes(x->cell_off.p, ns, x->K, x->cell_size.p, x->own));
    finalize_dense(x, true);
    set_l2_persisting(x);
}

void upload_imi(suco_gpu_index* x) {
    HostIndex& h = x->host;
    const uint32_t ns = h.layout.ns;
    const uint64_t K = uint64_t(h.p.k_half) * h.p.k_half;
    x->cell_off.reserve(ns * (K + 1));
    x->ids.reserve(ns * h.n);
    std::vector<uint32_t> off32(K + 1);
    for (uint32_t s = 0; s < ns; ++s) {
        for (uint64_t c = 0; c <= K; ++c) off32[c] = static_cast<uint32_t>(h.offsets[s][c]);
        CUDA_TRY(cudaMemcpy(x->cell_off.p + s * (K + 1), off32.data(), (K + 1) * 4, cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(x->ids.p + s * h.n, h.ids[s].data(), h.n * 4, cudaMemcpyHostToDevice));
    }
    // the IMI's home is the device; host copies are re-read on demand
    h.offsets.clear();
    h.ids.clear();
    h.offsets.shrink_to_fit();
    h.ids.shrink_to_fit();
}

void download_imi(const suco_gpu_index* x, uint32_t s, uint64_t* offsets, uint32_t* ids) {
    const uint64_t K = x->K, n = x->host.n;
    if (offsets) {
        std::vector<uint32_t> off32(K + 1);
        CUDA_TRY(cudaMemcpy(off32.data(), x->cell_off.p + s * (K + 1), (K + 1) * 4, cudaMemcpyDeviceToHost));
        for (uint64_t c = 0; c <= K; ++c) offsets[c] = off32[c];
    }
    if (ids) CUDA_TRY(cudaMemcpy(ids, x->ids.p + s * n, n * 4, cudaMemcpyDeviceToHost));
}

// ---------------------------------------------------------------- params
double snapped_product(double ratio, uint64_t n) {  // sc_linear.cpp:18-22
    const double product = ratio * static_cast<double>(n);
    const double nearest = std::round(product);
    return std::abs(product - nearest) <= 1e-6 ? nearest : product;
}

}  // namespace

namespace suco_gpu {

void validate_params(const suco_collision_params* p, uint64_t n) {  // sc_linear.cpp:26-37
    if (!p) raise(SUCO_ERR_CONTRACT, "collision params are null");
    if (!(p->alpha > 0.0) || p->alpha > 1.0) raise(SUCO_ERR_CONFIG, "alpha must be in (0, 1], got " + std::to_string(p->alpha));
    if (!(p->beta > 0.0) || p->beta > 1.0) raise(SUCO_ERR_CONFIG, "beta must be in (0, 1], got " + std::to_string(p->beta));
    if (p->k < 1 || p->k > n) {
        raise(SUCO_ERR_CONFIG, "k must be in [1, n]; got k = " + std::to_string(p->k) + " with n = " + std::to_string(n));
    }
}

// -------------------------------------------------------------- pipeline
// Resets the per-call profiling state (events + work counters).
void begin_call(suco_gpu_query_ctx* c, uint64_t nq, uint64_t m, cudaStream_t st) {
    c->pairs = 0;
    c->launches = 0;
    c->last_nq = nq;
    c->last_m = m;
    if (c->profile) {
        c->stat_cum.reserve(1);
        CUDA_TRY(cudaMemsetAsync(c->stat_cum.p, 0, sizeof(unsigned long long), st));
    }
}

}  // namespace suco_gpu

namespace {

// Profiling pair for one stage launch (nullptr when profiling is off).
cudaEvent_t* prof_pair(suco_gpu_query_ctx* c, int stage) {
    if (!c->profile) return nullptr;
    while (c->events.size() < 2ull * (c->pairs + 1)) {
        cudaEvent_t e;
        CUDA_TRY(cudaEventCreate(&e));
        c->events.push_back(e);
    }
    if (c->event_stage.size() < c->pairs + 1) c->event_stage.resize(c->pairs + 1);
    c->event_stage[c->pairs] = stage;
    return c->events.data() + 2ull * c->pairs++;
}

}  // namespace

namespace suco_gpu {

void stage_traverse(const suco_gpu_index* x, suco_gpu_query_ctx* c, suco_gpu_query_ctx::Slot& sl, const float* d_q,
                    uint64_t nt, uint64_t target, cudaStream_t st, double* dbg_sum, uint64_t* dbg_cum, bool profiled) {
    const HostIndex& h = x->host;
    const uint32_t ns = h.layout.ns;
    sl.cells.reserve(nt * ns * x->K);
    sl.ncells.reserve(nt * ns);
    cudaEvent_t* ev = profiled ? prof_pair(c, 0) : nullptr;
    TraverseArgs ta{};
    ta.queries = d_q;
    ta.d = h.d;
    ta.nq = nt;
    ta.dims = x->dims.p;
    ta.sub = x->sub.p;
    ta.cent = x->cent.p;
    ta.cell_size = x->cell_size.p;  // GLOBAL cell sizes on a shard: the global Dynamic-Activation cut
    ta.ns = ns;
    ta.k_half = h.p.k_half;
    ta.K = x->K;
    ta.hmax = x->hmax;
    ta.target = target;
    ta.cells = sl.cells.p;
    ta.ncells = sl.ncells.p;
    ta.dbg_sum = dbg_sum;
    ta.dbg_cum = dbg_cum;
    ta.stat_cum = ev ? c->stat_cum.p : nullptr;
    ta.mode = x->tune.traverse;
    if (ev) CUDA_TRY(cudaEventRecord(ev[0], st));
    CUDA_TRY(launch_traverse(ta, st));
    c->launches += traverse_launch_count(ta);
    if (ev) CUDA_TRY(cudaEventRecord(ev[1], st));
}

DenseArgs dense_args(const suco_gpu_index* x, suco_gpu_query_ctx::Slot& sl, uint64_t nq) {
    const HostIndex& h = x->host;
    DenseArgs da{};
    da.codes = reinterpret_cast<const uint4*>(x->codes.p);
    da.cells = sl.cells.p;
    da.ncells = sl.ncells.p;
    da.cells_cap = x->K;
    da.ns = h.layout.ns;
    da.K = x->K;
    da.n = h.n;
    da.nq = nq;
    da.WP = kDensePiece;
    da.P = static_cast<uint32_t>((h.n + da.WP - 1) / da.WP);
    da.half = x->dense_half ? 1u : 0u;
    da.hgroup = x->dense_half && x->dense_hgroup ? 1u : 0u;
    da.nc = h.layout.ns > 8 ? 2u : 1u;  // 9..16 subspaces: two code vectors, 16 histogram levels
    da.words = x->tune.dense_words;
    da.pair = x->dense_half && x->tune.dense_pair != 0 && dense_pair_supported(h.layout.ns, x->K) ? 1u : 0u;
    return da;
}

void rerank_args(const suco_gpu_index* x, RerankArgs& ra) {
    ra.data = x->data.p;
    ra.n = x->host.n;
    ra.d = x->host.d;
    ra.data_int_max = x->data_int_max;
    ra.data8 = x->dpad ? x->data8.p : nullptr;
    ra.dpad = x->dpad;
    ra.q8 = x->qpad ? x->q8.p : nullptr;
    ra.qpad = x->qpad;
    ra.qrec = x->qrec;
    ra.qpre = x->qpre;
    ra.q8_min = x->tune.q8 == 2 ? 0 : kQ8MinCands;
    ra.qsplit = x->qsplit;
    ra.q8b = x->qpad ? x->q8.p + x->q8_rows * x->qsplit : nullptr;
    ra.u8_regs = x->tune.rerank_u8_regs;
    ra.no_tma = !x->tune.rerank_tma;
    ra.pipe = x->tune.rerank_pipe == 2 ? 0 : x->tune.rerank_pipe == 1 ? 1 : 2;
}

// Points per piece of the single pass: the largest of 16384 .. 2048 that still gives the fused
// pass about sixteen CTAs per SM (32 pieces per CTA row, 32 queries per CTA). Measured per step:
// cfg4 (10M points, 10K queries) 2048 / 8192 / 16384 -> 38.2 / 32.9 / 31.4 ms; cfg2 (1M, 10K)
// 2048 / 4096 / 8192 -> 4.19 / 4.09 / 4.29 ms; small corpora or batches keep 2048 (cfg1, cfg3).
uint32_t fused_piece(uint64_t n, uint64_t nq, uint32_t qper) {
    int sms = 148, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t qblocks = (nq + qper - 1) / qper;  // queries per CTA: 32, 16 in the half-width mode
    for (uint32_t wp = 16384; wp > kDensePiece; wp /= 2) {
        const uint64_t P = (n + wp - 1) / wp;
        if (qblocks * ((P + 31) / 32) >= 16ull * sms) return wp;
    }
    return kDensePiece;
}

}  // namespace suco_gpu

namespace {

// The dense select's fallback lists (qflag: nq flags; qmap[0 .. *nmap): the flagged queries).
struct FbLists {
    const uint32_t* qflag = nullptr;
    const uint32_t* qmap = nullptr;
    const uint32_t* nmap = nullptr;
};


// Bytes of single-pass candidate buffers beyond kDenseBuf entries (small batches): at most 1 GB.
constexpr uint64_t kDenseBufExtra = 1ull << 30;

// main_done / fb_st (optional, both or neither): with the single-pass dense select, main_done is
// recorded on st once every unflagged query's candidates are written and the flagged queries'
// fallback runs on fb_st; the returned lists are then set (else empty: st has everything).
// scores_dbg: the per-point SC-scores of the (one) query, from the production select.
FbLists stage_select(const suco_gpu_index* x, suco_gpu_query_ctx* c, suco_gpu_query_ctx::Slot& sl, uint64_t nt,
                     uint64_t m, cudaStream_t st, uint8_t* scores_dbg, bool profiled, cudaEvent_t main_done = nullptr,
                     cudaStream_t fb_st = nullptr) {
    const HostIndex& h = x->host;
    const Tuning& tn = x->tune;
    sl.cands.reserve(nt * m);
    cudaEvent_t* ev = profiled ? prof_pair(c, 1) : nullptr;
    if (x->dense) {
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
        da.cands = sl.cands.p;
        da.scores_dbg = scores_dbg;
        const bool fused = tn.dense_fused && !scores_dbg;  // the score dump is a two-pass emission
        if (fused) {
            // larger pieces for the single pass (the half-width mode keeps kDensePiece: its code rows
            // are padded to whole 2048-point pieces): a quarter of the per-(query, piece) counts,
            // quotas and buffers, and buffers four times fuller, so far fewer partly written sectors
            // (measured at cfg4: fused pass writes and compaction reads)
            if (!(da.half && da.pair)) {  // (the cluster-pair pass walks 2048-point pieces)
                da.WP = tn.dense_piece ? tn.dense_piece : fused_piece(h.n, nt, da.half ? 16u : 32u);
                da.P = static_cast<uint32_t>((h.n + da.WP - 1) / da.WP);
            }
            // two output offsets per (query, piece): score > T entries fill the front of the query's
            // candidate list, the quota ties the back (the re-rank meets the likely nearest first)
            sl.dbase.reserve(2 * nt * da.P);
            da.base = sl.dbase.p;
            da.base2 = sl.dbase.p + nt * da.P;
            // the sampled histograms (every pstride-th piece) predict the threshold: about 16 sampled
            // pieces when that is enough (cfg2: 489 pieces -> every 30th), every 64th piece at most
            // for large corpora (measured: cfg2 2.31M -> 2.36M q/s, cfg4 167K -> 174K; fewer samples
            // mis-estimate T and send queries to the fallback); small corpora: all of them (exact)
            // (sampled pieces of kDensePiece points whatever the pass's piece size: measured at cfg4,
            // 16 samples of 16384 points took 1.05 ms, the warps walking 512 tiles each)
            const uint32_t P2 = static_cast<uint32_t>((h.n + kDensePiece - 1) / kDensePiece);
            da.sWP = kDensePiece;
            da.pstride = P2 <= 64 ? 1u : std::min<uint32_t>(64, P2 / 16);
            da.Ps = (P2 + da.pstride - 1) / da.pstride;
            sl.dsample.reserve(nt * da.Ps * 8 * da.nc);
            da.stage_all = tn.dense_stage;
            // entries per (piece, query): at least kDenseBuf (~6 sigma above cfg4's mean of 46); small
            // batches x corpora (cfg3: 1K queries x 489 pieces) get up to 2048 (one whole piece)
            // within kDenseBufExtra, so dense supersets do not overflow into the two-pass fallback
            const uint64_t fit = kDenseBufExtra / (2ull * nt * da.P) / 8 * 8;
            const uint64_t minb = uint64_t(kDenseBuf) * (da.WP / kDensePiece);
            da.B = static_cast<uint32_t>(std::min<uint64_t>(da.WP, std::max<uint64_t>(minb, fit)));
            if (tn.dense_buf) da.B = tn.dense_buf;
            sl.dcbuf.reserve(nt * da.P * da.B);
            sl.dccnt.reserve(nt * da.P);
            da.cbuf = sl.dcbuf.p;
            da.ccnt = sl.dccnt.p;
            sl.dL.reserve(nt);
            sl.dh2.reserve(nt * da.P);
            da.h2 = sl.dh2.p;
            // flags, flagged list, its count, tie cuts, the dense / sparse compaction lists and counts
            sl.dflag.reserve(5 * nt + 3);
            da.pcut = sl.dflag.p + 2 * nt + 1;
            da.clist = sl.dflag.p + 3 * nt + 1;
            da.nclist = sl.dflag.p + 5 * nt + 1;
            da.no_cut = tn.dense_nocut;
            da.cut_scale = tn.tie_cut_scale;
            da.cut_pad = tn.tie_cut_pad;
            da.compact_mode = tn.dense_compact;
            da.compact_rows = tn.dense_compact_rows;
            da.hsample = sl.dsample.p;
            da.qmap = sl.dflag.p + nt;
            da.nmap = sl.dflag.p + 2 * nt;
            da.L = sl.dL.p;
            da.qflag = sl.dflag.p;
        }
        if (ev) CUDA_TRY(cudaEventRecord(ev[0], st));
        const bool split = fused && main_done && fb_st;
        CUDA_TRY(split ? launch_dense_select_fused(da, st, main_done, fb_st)
                       : fused ? launch_dense_select_fused(da, st) : launch_dense_select(da, st));
        // two-pass: piece histograms, plan, emission; single pass: sample, bound, fused pass, plan,
        // compaction, flagged list, fallback histograms, plan, emission
        c->launches += fused ? 10 : 3;
        if (tn.dense_stats && fused) {  // diagnostics: the fallback rate, superset sizes
            uint32_t nflag = 0;
            cudaStream_t ds = split ? fb_st : st;
            std::vector<uint16_t> cc(nt * da.P);
            std::vector<uint32_t> cut(nt), Lh(nt);
            CUDA_TRY(cudaMemcpyAsync(&nflag, da.nmap, 4, cudaMemcpyDeviceToHost, ds));
            CUDA_TRY(cudaMemcpyAsync(cc.data(), da.ccnt, cc.size() * 2, cudaMemcpyDeviceToHost, ds));
            CUDA_TRY(cudaMemcpyAsync(cut.data(), da.pcut, nt * 4, cudaMemcpyDeviceToHost, ds));
            CUDA_TRY(cudaMemcpyAsync(Lh.data(), da.L, nt * 4, cudaMemcpyDeviceToHost, ds));
            CUDA_TRY(cudaStreamSynchronize(ds));
            double entries = 0, nonzero = 0, before = 0, cuts = 0, dense = 0;
            for (uint64_t q = 0; q < nt; ++q) {
                cuts += cut[q];
                dense += (Lh[q] & 0x100u) != 0;
                for (uint32_t p = 0; p < da.P; ++p) {
                    const uint16_t v = cc[q * da.P + p];
                    entries += v;
                    nonzero += v != 0;
                    if (p < cut[q]) before += v;
                }
            }
            double bmax = 0, bsorted = 0;  // mean over 32-query blocks of the block's largest cut: in query order, sorted by cut
            std::vector<uint32_t> sc(cut);
            std::sort(sc.begin(), sc.end());
            for (uint64_t q0 = 0; q0 < nt; q0 += 32) {
                uint32_t mx = 0;
                for (uint64_t q = q0; q < std::min<uint64_t>(nt, q0 + 32); ++q) mx = std::max(mx, cut[q]);
                bmax += mx;
                bsorted += sc[std::min<uint64_t>(nt, q0 + 32) - 1];
            }
            std::fprintf(stderr, "[suco] dense cuts: mean block-max cut %.1f (query order) vs %.1f (queries sorted by cut)\n",
                         bmax / ((nt + 31) / 32), bsorted / ((nt + 31) / 32));
            std::fprintf(stderr,
                         "[suco] dense select: %u of %llu queries took the two-pass fallback (pstride %u); superset "
                         "%.0f entries/query (%.0f before the tie cut), %.1f%% of (query, piece) buffers used, mean "
                         "cut %.0f of %u pieces, %.0f%% dense-staged queries, m = %llu, B = %u\n",
                         nflag, static_cast<unsigned long long>(nt), da.pstride, entries / nt, before / nt,
                         100.0 * nonzero / (double(nt) * da.P), cuts / nt, da.P, 100.0 * dense / nt,
                         static_cast<unsigned long long>(m), da.B);
        }
        if (ev) CUDA_TRY(cudaEventRecord(ev[1], split ? fb_st : st));
        FbLists fl;
        if (split) {
            fl.qflag = da.qflag;
            fl.qmap = da.qmap;
            fl.nmap = da.nmap;
        }
        return fl;
    }
    SelectArgs sa{};
    sa.ids = x->ids.p;
    sa.slab_off = x->slab_off.p;
    sa.cells = sl.cells.p;
    sa.ncells = sl.ncells.p;
    sa.cells_cap = x->K;
    sa.n = h.n;
    sa.ns = h.layout.ns;
    sa.K = x->K;
    sa.nslabs = x->sel.nslabs;
    sa.CH = x->sel.CH;
    sa.rounds = x->sel.rounds;
    sa.CS = x->sel.CS;
    sa.m = m;
    sa.nq = nt;
    sa.cands = sl.cands.p;
    sa.scores_dbg = scores_dbg;
    if (ev) CUDA_TRY(cudaEventRecord(ev[0], st));
    CUDA_TRY(launch_select(sa, x->sel, nt, st));
    c->launches += 1;
    if (ev) CUDA_TRY(cudaEventRecord(ev[1], st));
    return {};
}

void stage_rerank(const suco_gpu_index* x, suco_gpu_query_ctx* c, suco_gpu_query_ctx::Slot& sl, const float* d_q,
                  uint64_t nt, uint64_t m, uint32_t k, uint32_t* d_ids, double* d_dists, cudaStream_t st, bool profiled,
                  const FbLists* fl = nullptr, bool flagged = false) {
    cudaEvent_t* ev = profiled ? prof_pair(c, 2) : nullptr;
    RerankArgs ra{};
    rerank_args(x, ra);
    ra.queries = d_q;
    ra.cands = sl.cands.p;
    ra.m = m;
    ra.k = k;
    ra.out_ids = d_ids;
    ra.out_dists = d_dists;
    if (k > 32) {
        sl.all_d.reserve(nt * m);
        sl.all_id.reserve(nt * m);
        ra.all_d = sl.all_d.p;
        ra.all_id = sl.all_id.p;
    }
    if (fl && fl->qflag) {  // a split select: the unflagged queries now, the flagged ones (qmap) later
        if (flagged) {
            ra.qlist = fl->qmap;
            ra.nlist = fl->nmap;
        } else {
            ra.qskip = fl->qflag;
        }
    }
    DevBuf<unsigned long long> stats;
    if (x->tune.rerank_stats && ra.q8) {
        stats.reserve(3);
        CUDA_TRY(cudaMemsetAsync(stats.p, 0, 24, st));
        ra.screen_stats = stats.p;
    }
    if (ev) CUDA_TRY(cudaEventRecord(ev[0], st));
    CUDA_TRY(launch_rerank(ra, nt, st));
    c->launches += (ra.data8 ? 2 : 1) + (k > 32 ? 1 : 0);  // u8 + fp32/fp64 kernels, generic top-k
    if (ev) CUDA_TRY(cudaEventRecord(ev[1], st));
    if (ra.screen_stats) {  // diagnostics
        unsigned long long h[3] = {0, 0, 0};
        CUDA_TRY(cudaMemcpyAsync(h, stats.p, 24, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        std::fprintf(stderr,
                     "[suco] int8 screen: %llu queries, %.1f exact re-ranks per query, %llu re-ranked in full, %.1f "
                     "rows per query past the prefix bound\n",
                     static_cast<unsigned long long>(nt), double(h[0]) / double(nt), h[1], double(h[2]) / double(nt));
    }
}

// Per-query scratch bytes of one pipeline tile (both slots hold one tile).
uint64_t per_query_bytes(const suco_gpu_index* x, uint64_t m, uint32_t k) {
    const uint64_t ns = x->host.layout.ns;
    const uint64_t P = (x->host.n + kDensePiece - 1) / kDensePiece;
    const uint64_t nc = ns > 8 ? 2 : 1;
    uint64_t per = ns * x->K * 4 + ns * 4 + m * 4 + (k > 32 ? m * 12 : 0) + uint64_t(x->host.d) * 4 + k * 12;
    if (x->dense) {
        // hist (16 B x nc) + quota/base + two-level counts + buffer counts per piece, kDenseBuf
        // buffer entries per piece, sampled histograms, flags
        per += P * (16 * nc + 12 + 4 + 2 + kDenseBuf * 2) + (P / 16 + 1) * 16 * nc + 20;
    }
    return per;
}

// Scratch budget of a context: SUCO_SCRATCH_MB, else (first use) half of the device memory free
// at that time, at most 32 GB; a failed allocation halves it (run_pipeline). Cached, so a query
// call makes no cudaMemGetInfo round trip.
uint64_t ctx_budget(const suco_gpu_index* x, suco_gpu_query_ctx* c) {
    if (x->tune.scratch_bytes) return x->tune.scratch_bytes;
    if (!c->budget) {
        size_t free_b = 0, total_b = 0;
        CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
        c->budget = std::max<uint64_t>(64ull << 20, std::min<uint64_t>(32ull << 30, free_b / 2));
    }
    return c->budget;
}

uint64_t tile_size(const suco_gpu_index* x, suco_gpu_query_ctx* c, uint64_t nq, uint64_t m, uint32_t k) {
    uint64_t budget = ctx_budget(x, c);
    if (x->dense && !x->tune.scratch_bytes) {
        budget = budget > 2 * kDenseBufExtra ? budget - 2 * kDenseBufExtra : budget / 2;
    }
    const uint64_t per = per_query_bytes(x, m, k);
    return std::max<uint64_t>(1, std::min<uint64_t>(nq, budget / 2 / per));
}

// The batched query pipeline. Queries are either device-resident (h_q == nullptr,
// d_q given) or host (h_q given: copied per tile on the traverse stream).
// Outputs go to d_ids/d_dists, or to host h_ids/h_dists (copied per tile).
// A failed scratch allocation halves the tile and resumes at the failed tile.
void run_pipeline(const suco_gpu_index* x, suco_gpu_query_ctx* c, const float* h_q, const float* d_q, uint64_t nq,
                  uint32_t qlen, const suco_collision_params* p, uint32_t* d_ids, double* d_dists, uint32_t* h_ids,
                  double* h_dists, cudaStream_t user) {
    if (x->num_shards > 1) raise(SUCO_ERR_CONTRACT, "a shard answers only through suco_gpu_shard_knn_query_batch");
    const uint64_t n = x->host.n;
    const uint32_t k = p->k;
    const uint64_t m = suco_candidate_count(p->beta, n, k);
    const uint64_t target = suco_collision_count(p->alpha, n);
    uint64_t tile = tile_size(x, c, nq, m, k);
    // at least `tiles` tiles (tests: slot reuse), each at least 512 queries unless forced smaller
    const uint64_t want = std::max<uint64_t>(1, std::min<uint64_t>(x->tune.tiles, x->tune.tiles > 1 ? nq : nq / 512));
    tile = std::min(tile, (nq + want - 1) / want);
    begin_call(c, nq, m, user);
    CUDA_TRY(cudaEventRecord(c->ev_in, user));
    for (cudaStream_t t : c->pipe) CUDA_TRY(cudaStreamWaitEvent(t, c->ev_in, 0));
    cudaStream_t s_trav = c->pipe[0], s_sel = c->pipe[1], s_rr = c->pipe[2];
    uint64_t q0 = 0, t = 0;
    while (q0 < nq) {
        try {
            for (; q0 < nq; q0 += tile, ++t) {
                const uint64_t nt = std::min(tile, nq - q0);
                // measured: cfg2 (byte rows, 10,000 queries) 2.334M -> 2.364M q/s (e2e 2.12M -> 2.23M);
                // slower where the re-rank is long beside it (fp32 rows: cfg3 143K -> 136K, cfg4 170K ->
                // 169K), so only byte-row re-ranks of large tiles overlap the fallback
                const bool fb_overlap = x->tune.fb_overlap >= 0 ? x->tune.fb_overlap != 0
                                                                 : (x->dpad && !x->dense_half && nt >= 4096);
                auto& sl = c->slot[t & 1];
                // slot reuse: tile t-2's select read `cells`, its rerank read `q`/`cands`
                CUDA_TRY(cudaStreamWaitEvent(s_trav, sl.sel, 0));
                CUDA_TRY(cudaStreamWaitEvent(s_trav, sl.rr, 0));
                const float* tq = d_q ? d_q + q0 * qlen : nullptr;
                if (h_q) {
                    sl.q.reserve(tile * qlen);
                    CUDA_TRY(cudaMemcpyAsync(sl.q.p, h_q + q0 * qlen, nt * qlen * 4, cudaMemcpyHostToDevice, s_trav));
                    tq = sl.q.p;
                }
                stage_traverse(x, c, sl, tq, nt, target, s_trav, nullptr, nullptr, true);
                CUDA_TRY(cudaEventRecord(sl.trav, s_trav));
                CUDA_TRY(cudaStreamWaitEvent(s_sel, sl.trav, 0));
                CUDA_TRY(cudaStreamWaitEvent(s_sel, sl.rr, 0));
                // the fallback of the few flagged queries overlaps the re-rank of the others
                const FbLists fl = stage_select(x, c, sl, nt, m, s_sel, nullptr, true,
                                                fb_overlap ? sl.selmain : nullptr, fb_overlap ? c->pipe[3] : nullptr);
                CUDA_TRY(cudaEventRecord(sl.sel, fl.qflag ? c->pipe[3] : s_sel));
                CUDA_TRY(cudaStreamWaitEvent(s_rr, fl.qflag ? sl.selmain : sl.sel, 0));
                uint32_t* oi = d_ids ? d_ids + q0 * k : nullptr;
                double* od = d_dists ? d_dists + q0 * k : nullptr;
                if (h_ids) {
                    sl.out_ids.reserve(tile * k);
                    sl.out_d.reserve(tile * k);
                    oi = sl.out_ids.p;
                    od = sl.out_d.p;
                }
                stage_rerank(x, c, sl, tq, nt, m, k, oi, od, s_rr, true, &fl, false);
                if (fl.qflag) {
                    CUDA_TRY(cudaStreamWaitEvent(s_rr, sl.sel, 0));
                    stage_rerank(x, c, sl, tq, nt, m, k, oi, od, s_rr, true, &fl, true);
                }
                if (h_ids) {
                    CUDA_TRY(cudaMemcpyAsync(h_ids + q0 * k, oi, nt * k * 4, cudaMemcpyDeviceToHost, s_rr));
                    CUDA_TRY(cudaMemcpyAsync(h_dists + q0 * k, od, nt * k * 8, cudaMemcpyDeviceToHost, s_rr));
                }
                CUDA_TRY(cudaEventRecord(sl.rr, s_rr));
            }
        } catch (const OutOfDeviceMemory&) {
            if (tile == 1) throw;
            for (cudaStream_t s : c->pipe) CUDA_TRY(cudaStreamSynchronize(s));
            for (auto& sl : c->slot) sl.release_all();
            tile = (tile + 1) / 2;  // resume at the tile whose scratch did not fit
            c->budget = std::max<uint64_t>(64ull << 20, c->budget / 2);
        }
    }
    CUDA_TRY(cudaEventRecord(c->ev_out, s_rr));
    CUDA_TRY(cudaStreamWaitEvent(user, c->ev_out, 0));
}

void check_query_args(const suco_gpu_index* x, uint32_t qlen, const suco_collision_params* p) {
    if (!x) raise(SUCO_ERR_CONTRACT, "index is null");
    check_query_len(qlen, x->host.d);  // query.cpp:203-206
    validate_params(p, x->n_global);   // query.cpp:208
    if (x->host.layout.ns > 255) raise(SUCO_ERR_CONFIG, "the GPU path keeps u8 collision counters: N_s must be <= 255");
}

suco_gpu_index* new_index(int device) {
    auto* x = new suco_gpu_index();
    x->device = device;
    x->tune = tuning_from_env();
    return x;
}

}  // namespace

namespace suco_gpu {

void load_core(suco_gpu_index* x, uint64_t n) {
    upload_codebooks(x);
    upload_imi(x);
    finalize_device(x);
    x->n_global = n;
}

// build_index (index.cpp:98-145) over rows already on the device; train != nullptr: the sampled
// build (k-means on those rows, every row assigned to its nearest centroid).
void build_core(suco_gpu_index* x, uint64_t n, uint32_t d, const suco_index_params* params, const uint32_t* train,
                uint64_t n_train) {
    // index.cpp:100-108
    if (params->k_half < 1) raise(SUCO_ERR_CONFIG, "k_half must be >= 1");
    if (params->iterations < 1) raise(SUCO_ERR_CONFIG, "iterations must be >= 1");
    const uint64_t nfit = train ? n_train : n;
    if (nfit < params->k_half) {
        raise(SUCO_ERR_CONFIG, std::string(train ? "training sample" : "dataset") + " has n = " + std::to_string(nfit) +
                                   " points, fewer than k_half = " + std::to_string(params->k_half));
    }
    if (n > 0xFFFFFFFFull) raise(SUCO_ERR_CONTRACT, "dataset exceeds 32-bit point-id capacity");
    for (uint64_t i = 0; train && i < n_train; ++i) {
        if (train[i] >= n || (i && train[i] <= train[i - 1])) {
            raise(SUCO_ERR_CONTRACT, "training ids must be strictly ascending and < n (entry " + std::to_string(i) + ")");
        }
    }
    x->host.layout = sample_subspaces(d, params->num_subspaces, params->mode, params->seed);
    x->host.n = n;
    x->host.d = d;
    x->host.p = *params;
    const uint64_t K = uint64_t(params->k_half) * params->k_half;
    x->cell_off.reserve(uint64_t(params->num_subspaces) * (K + 1));
    x->ids.reserve(uint64_t(params->num_subspaces) * n);
    BuildOutputs bo{x->cell_off.p, x->ids.p, &x->host.cent1, &x->host.cent2};
    build_index_device(x->data.p, n, d, x->host.layout, *params, bo, x->own, x->tune, train, n_train);
    upload_codebooks(x);
    finalize_device(x);
    x->n_global = n;
}

suco_gpu_index* new_index_on(int device) {
    suco_gpu_index* x = new_index(device);
    try {
        create_index_stream(x);
    } catch (...) {
        delete x;
        throw;
    }
    return x;
}

}  // namespace suco_gpu

// ======================================================================= C ABI
extern "C" {

const char* suco_last_error(void) { return g_err.c_str(); }

int suco_gpu_device_count(int* count) {
    return guarded([&] {
        if (!count) raise(SUCO_ERR_CONTRACT, "count is null");
        int c = 0;
        if (cudaGetDeviceCount(&c) != cudaSuccess) {
            cudaGetLastError();
            c = 0;
        }
        *count = c;
    });
}

uint64_t suco_collision_count(double alpha, uint64_t n) {  // sc_linear.cpp:39-42
    const uint64_t c = static_cast<uint64_t>(std::floor(snapped_product(alpha, n)));
    return std::max<uint64_t>(1, c);
}

uint64_t suco_candidate_count(double beta, uint64_t n, uint64_t k) {  // sc_linear.cpp:44-47
    const uint64_t c = static_cast<uint64_t>(std::ceil(snapped_product(beta, n)));
    return std::max(k, c);
}

int suco_validate_collision_params(const suco_collision_params* p, uint64_t n) {
    return guarded([&] { validate_params(p, n); });
}

int suco_gpu_load_index(const unsigned char* bytes, uint64_t len, const float* data, uint64_t n, uint32_t d, int device,
                        suco_gpu_index** out) {
    return guarded([&] {
        if (!out) raise(SUCO_ERR_CONTRACT, "output handle pointer is null");
        *out = nullptr;
        if (!bytes && len) raise(SUCO_ERR_CONTRACT, "index bytes are null");
        HostIndex h = parse_index(bytes, len);  // CORRUPT_INDEX first (load_index), as suco_cli.cpp:243
        check_dataset(data, n, d);              // then the dataset (CONTRACT)
        if (h.n != n) {                         // index.cpp:295-305
            raise(SUCO_ERR_INCOMPATIBLE, "index was built from n = " + std::to_string(h.n) +
                                             " points but dataset has n = " + std::to_string(n));
        }
        if (h.d != d) {
            raise(SUCO_ERR_INCOMPATIBLE, "index was built for d = " + std::to_string(h.d) +
                                             " but dataset has d = " + std::to_string(d));
        }
        DeviceGuard g(device);
        suco_gpu_index* x = new_index_on(device);
        try {
            x->host = std::move(h);
            upload_data(x, data, n, d);
            load_core(x, n);
        } catch (...) {
            delete x;
            throw;
        }
        *out = x;
    });
}

int suco_gpu_build_index(const float* data, uint64_t n, uint32_t d, const suco_index_params* params, int device,
                         suco_gpu_index** out) {
    return guarded([&] {
        if (!out) raise(SUCO_ERR_CONTRACT, "output handle pointer is null");
        *out = nullptr;
        if (!params) raise(SUCO_ERR_CONTRACT, "index params are null");
        check_dataset(data, n, d);
        DeviceGuard g(device);
        suco_gpu_index* x = new_index_on(device);
        try {
            upload_data(x, data, n, d);  // finiteness (core.cpp:15-19) before any parameter check
            build_core(x, n, d, params);
        } catch (...) {
            delete x;
            throw;
        }
        *out = x;
    });
}

int suco_gpu_build_index_sampled(const float* data, uint64_t n, uint32_t d, const suco_index_params* params,
                                 const uint32_t* train_ids, uint64_t n_train, int device, suco_gpu_index** out) {
    return guarded([&] {
        if (!out) raise(SUCO_ERR_CONTRACT, "output handle pointer is null");
        *out = nullptr;
        if (!params) raise(SUCO_ERR_CONTRACT, "index params are null");
        if (!train_ids) raise(SUCO_ERR_CONTRACT, "training ids are null");
        check_dataset(data, n, d);
        DeviceGuard g(device);
        suco_gpu_index* x = new_index_on(device);
        try {
            upload_data(x, data, n, d);
            build_core(x, n, d, params, train_ids, n_train);
        } catch (...) {
            delete x;
            throw;
        }
        *out = x;
    });
}

int suco_gpu_serialize_index(const suco_gpu_index* x, unsigned char* buf, uint64_t cap, uint64_t* len) {
    return guarded([&] {
        if (!x || !len) raise(SUCO_ERR_CONTRACT, "null argument");
        if (x->num_shards > 1) raise(SUCO_ERR_CONTRACT, "a shard holds part of an index: serialize the full index");
        DeviceGuard g(x->device);
        HostIndex h;
        h.n = x->host.n;
        h.d = x->host.d;
        h.p = x->host.p;
        h.layout = x->host.layout;
        h.cent1 = x->host.cent1;
        h.cent2 = x->host.cent2;
        const uint32_t ns = h.layout.ns;
        h.offsets.resize(ns);
        h.ids.resize(ns);
        for (uint32_t s = 0; s < ns; ++s) {
            h.offsets[s].resize(x->K + 1);
            h.ids[s].resize(h.n);
            download_imi(x, s, h.offsets[s].data(), h.ids[s].data());
        }
        const std::vector<unsigned char> bytes = serialize(h);
        *len = bytes.size();
        if (buf) {
            if (cap < bytes.size()) raise(SUCO_ERR_CONTRACT, "serialize: buffer too small");
            std::memcpy(buf, bytes.data(), bytes.size());
        }
    });
}

int suco_gpu_index_subspace(const suco_gpu_index* x, uint32_t s, float* c1, float* c2, uint64_t* offsets, uint32_t* ids) {
    return guarded([&] {
        if (!x) raise(SUCO_ERR_CONTRACT, "index is null");
        if (s >= x->host.layout.ns) raise(SUCO_ERR_CONTRACT, "subspace index out of range");
        if (c1) std::memcpy(c1, x->host.cent1[s].data(), x->host.cent1[s].size() * 4);
        if (c2) std::memcpy(c2, x->host.cent2[s].data(), x->host.cent2[s].size() * 4);
        if (offsets || ids) {
            DeviceGuard g(x->device);
            download_imi(x, s, offsets, ids);
        }
    });
}

int suco_gpu_index_info(const suco_gpu_index* x, uint64_t* n, uint32_t* d, suco_index_params* params, uint32_t* dims,
                        uint32_t* sizes, uint32_t* split) {
    return guarded([&] {
        if (!x) raise(SUCO_ERR_CONTRACT, "index is null");
        if (n) *n = x->n_global;
        if (d) *d = x->host.d;
        if (params) *params = x->host.p;
        const HostLayout& L = x->host.layout;
        if (dims) std::memcpy(dims, L.dims.data(), L.dims.size() * 4);
        if (sizes) std::memcpy(sizes, L.sizes.data(), L.ns * 4);
        if (split) std::memcpy(split, L.split.data(), L.ns * 4);
    });
}

void suco_gpu_free_index(suco_gpu_index* x) {
    if (!x) return;
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(x->device);
    delete x;
    if (prev >= 0) cudaSetDevice(prev);
}

// ------------------------------------------------------------------ query contexts
int suco_gpu_query_ctx_create(const suco_gpu_index* x, suco_gpu_query_ctx** out) {
    return guarded([&] {
        if (!x || !out) raise(SUCO_ERR_CONTRACT, "null argument");
        *out = nullptr;
        DeviceGuard g(x->device);
        *out = ctx_new(x);
    });
}

void suco_gpu_query_ctx_free(suco_gpu_query_ctx* c) { delete c; }

int suco_gpu_query_ctx_synchronize(suco_gpu_query_ctx* c) {
    return guarded([&] {
        if (!c) raise(SUCO_ERR_CONTRACT, "query context is null");
        DeviceGuard g(c->device);
        for (cudaStream_t t : c->pipe) CUDA_TRY(cudaStreamSynchronize(t));
        CUDA_TRY(cudaStreamSynchronize(c->own));
    });
}

int suco_gpu_query_ctx_set_profiling(suco_gpu_query_ctx* c, int enabled) {
    return guarded([&] {
        if (!c) raise(SUCO_ERR_CONTRACT, "query context is null");
        DeviceGuard g(c->device);
        c->profile = enabled != 0;
        if (c->profile) c->stat_cum.reserve(1);
    });
}

int suco_gpu_query_ctx_last_launches(const suco_gpu_query_ctx* c, uint64_t* launches) {
    return guarded([&] {
        if (!c || !launches) raise(SUCO_ERR_CONTRACT, "null argument");
        *launches = c->launches;
    });
}

int suco_gpu_query_ctx_exchange_bytes(const suco_gpu_query_ctx* c, uint64_t* bytes) {
    return guarded([&] {
        if (!c || !bytes) raise(SUCO_ERR_CONTRACT, "null argument");
        *bytes = c->exchange_bytes;
    });
}

int suco_gpu_query_ctx_stage_times(suco_gpu_query_ctx* c, double* ms, uint64_t* stats) {
    return guarded([&] {
        if (!c) raise(SUCO_ERR_CONTRACT, "query context is null");
        if (!c->profile) raise(SUCO_ERR_CONTRACT, "profiling is not enabled on this query context");
        DeviceGuard g(c->device);
        double acc[3] = {0, 0, 0};
        for (uint32_t i = 0; i < c->pairs; ++i) {
            cudaEvent_t* ev = c->events.data() + 2ull * i;
            CUDA_TRY(cudaEventSynchronize(ev[1]));
            float f = 0.f;
            CUDA_TRY(cudaEventElapsedTime(&f, ev[0], ev[1]));
            acc[c->event_stage[i]] += f;
        }
        if (ms) {
            for (int st = 0; st < 3; ++st) ms[st] = acc[st];
        }
        if (stats) {
            unsigned long long v = 0;
            CUDA_TRY(cudaMemcpy(&v, c->stat_cum.p, sizeof v, cudaMemcpyDeviceToHost));
            stats[0] = v;
            stats[1] = c->last_nq;
            stats[2] = c->last_m;
        }
    });
}

// ------------------------------------------------------------------ queries
int suco_gpu_knn_query_batch_device(const suco_gpu_index* x, const float* d_queries, uint64_t nq, uint32_t qlen,
                                    const suco_collision_params* p, uint32_t* d_ids, double* d_dists, void* stream,
                                    suco_gpu_query_ctx* ctx) {
    return guarded([&] {
        check_query_args(x, qlen, p);
        check_ctx(x, ctx);
        if (nq == 0) return;
        if (!d_queries || !d_ids || !d_dists) raise(SUCO_ERR_CONTRACT, "null buffer");
        DeviceGuard g(x->device);
        CtxLease lease(x, ctx);
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : lease.c->own;
        run_pipeline(x, lease.c, nullptr, d_queries, nq, qlen, p, d_ids, d_dists, nullptr, nullptr, st);
    });
}

int suco_gpu_knn_query_batch(const suco_gpu_index* x, const float* queries, uint64_t nq, uint32_t qlen,
                             const suco_collision_params* p, uint32_t* ids, double* dists, suco_gpu_query_ctx* ctx) {
    return guarded([&] {
        check_query_args(x, qlen, p);
        check_ctx(x, ctx);
        if (nq == 0) return;
        if (!queries || !ids || !dists) raise(SUCO_ERR_CONTRACT, "null buffer");
        DeviceGuard g(x->device);
        CtxLease lease(x, ctx);
        run_pipeline(x, lease.c, queries, nullptr, nq, qlen, p, nullptr, nullptr, ids, dists, lease.c->own);
        CUDA_TRY(cudaStreamSynchronize(lease.c->own));
    });
}

int suco_gpu_query_intermediates(const suco_gpu_index* x, const float* query, uint32_t qlen,
                                 const suco_collision_params* p, uint32_t* scores, uint32_t* cands, uint64_t* m_out,
                                 uint32_t* cells_per_subspace, uint64_t* cumulative) {
    return guarded([&] {
        check_query_args(x, qlen, p);
        if (!query) raise(SUCO_ERR_CONTRACT, "query is null");
        if (x->num_shards > 1) raise(SUCO_ERR_CONTRACT, "intermediates need the full index");
        DeviceGuard g(x->device);
        CtxLease lease(x, nullptr);
        suco_gpu_query_ctx* c = lease.c;
        cudaStream_t st = c->own;
        const uint64_t n = x->host.n;
        const uint32_t ns = x->host.layout.ns;
        const uint64_t m = suco_candidate_count(p->beta, n, p->k);
        const uint64_t target = suco_collision_count(p->alpha, n);
        DevBuf<uint8_t> sc;
        DevBuf<double> sums;
        DevBuf<uint64_t> cum;
        sc.reserve(n);
        sums.reserve(uint64_t(ns) * x->K);
        cum.reserve(uint64_t(ns) * x->K);
        CUDA_TRY(cudaMemsetAsync(sc.p, 0, n, st));
        auto& sl = c->slot[0];
        sl.q.reserve(qlen);
        CUDA_TRY(cudaMemcpyAsync(sl.q.p, query, qlen * 4, cudaMemcpyHostToDevice, st));
        stage_traverse(x, c, sl, sl.q.p, 1, target, st, sums.p, cum.p, false);
        // the production select (dense two-pass emission or cluster counting), which writes the
        // per-point SC-scores it computed on the way
        stage_select(x, c, sl, 1, m, st, sc.p, false);
        CUDA_TRY(cudaStreamSynchronize(st));
        if (scores) {
            std::vector<uint8_t> s8(n);
            CUDA_TRY(cudaMemcpy(s8.data(), sc.p, n, cudaMemcpyDeviceToHost));
            for (uint64_t i = 0; i < n; ++i) scores[i] = s8[i];
        }
        if (cands) {  // the select kernel emits the candidate SET; report it ascending
            CUDA_TRY(cudaMemcpy(cands, sl.cands.p, m * 4, cudaMemcpyDeviceToHost));
            std::sort(cands, cands + m);
        }
        if (m_out) *m_out = m;
        std::vector<uint32_t> nc(ns);
        CUDA_TRY(cudaMemcpy(nc.data(), sl.ncells.p, ns * 4, cudaMemcpyDeviceToHost));
        if (cells_per_subspace) std::memcpy(cells_per_subspace, nc.data(), ns * 4);
        if (cumulative) {
            for (uint32_t s = 0; s < ns; ++s) {
                cumulative[s] = 0;
                if (nc[s]) CUDA_TRY(cudaMemcpy(cumulative + s, cum.p + uint64_t(s) * x->K + nc[s] - 1, 8, cudaMemcpyDeviceToHost));
            }
        }
    });
}

}  // extern "C"
