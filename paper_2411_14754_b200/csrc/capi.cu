// C-ABI implementation (include/suco_b200.h): validation in the reference's
// order, index upload/build, and the query pipeline
//   traverse (warp per query x subspace) -> select (cluster per query)
//   -> rerank (CTA per query)
// enqueued on the index's stream, tiled over the query batch so the
// per-query scratch (retrieved cells, candidates) stays bounded.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/suco_b200.h"
#include "build.h"
#include "index_format.h"
#include "kernels.h"

using namespace suco_gpu;

namespace {

thread_local std::string g_err;

#define CUDA_TRY(x)                                                                                     \
    do {                                                                                                \
        const cudaError_t e_ = (x);                                                                     \
        if (e_ != cudaSuccess) raise(SUCO_ERR_INTERNAL, std::string("CUDA error '") +                 \
                                                            cudaGetErrorString(e_) + "' in " #x);       \
    } while (0)

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return SUCO_OK;
    } catch (const Status& s) {
        g_err = s.msg;
        return s.code;
    } catch (const std::bad_alloc&) {
        g_err = "out of host memory";
        return SUCO_ERR_INTERNAL;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SUCO_ERR_INTERNAL;
    }
}

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t cap = 0;
    void reserve(size_t count) {
        if (count <= cap && p) return;
        release();
        CUDA_TRY(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
        cap = count;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    ~DevBuf() { release(); }
};

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
            cudaGetLastError();
            raise(SUCO_ERR_INTERNAL, "no CUDA device available: the SuCo B200 path has no CPU fallback");
        }
        if (dev < 0 || dev >= count) raise(SUCO_ERR_INTERNAL, "CUDA device " + std::to_string(dev) + " does not exist");
        CUDA_TRY(cudaGetDevice(&prev));
        if (prev != dev) CUDA_TRY(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

int cluster_size_from_env() {  // 0 = choose by occupancy (plan_select)
    const char* v = std::getenv("SUCO_CLUSTER");
    if (!v) return 0;
    const int c = std::atoi(v);
    return (c >= 1 && c <= 16) ? c : 0;
}

}  // namespace

struct suco_gpu_index {
    int device = 0;
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    HostIndex host;  // layout, params, centroids (IMI lives on the device)
    uint32_t K = 0, hmax = 0;
    DevBuf<float> data;
    DevBuf<uint32_t> dims;
    DevBuf<SubDesc> sub;
    DevBuf<float> cent;
    DevBuf<uint32_t> cell_off;   // ns x (K+1)
    DevBuf<uint32_t> cell_size;  // ns x K
    DevBuf<uint32_t> ids;        // ns x n
    DevBuf<uint32_t> slab_off;   // ns x K x (nslabs+1)
    SelectConfig sel{};
    float data_int_max = -1.f;  // integer certificate of the dataset (rerank fp32 path)
    DevBuf<uint8_t> data8;      // u8 copy of the rows when they are integers in [0, 255] (rerank u8 path)
    DevBuf<uint16_t> codes;     // n x 8: s*K + cell of every point (dense select, N_s <= 8)
    bool dense = false;         // select stage = dense bit-sliced 32-query blocks (dense.cu)
    bool dense_half = false;    // ... in the half-width mode (16-query blocks, u16 masks; large N_s*K)
    uint64_t phase1_nq = 0;     // shard: queries of the last dense phase 1 (phase 2 re-scores them)
    uint32_t dpad = 0;          // row bytes of data8 (0: no u8 copy)
    // block-cyclic shard (suco_gpu_make_shard): global blocks j with j % num_shards == shard
    uint32_t shard = 0, num_shards = 1, block = 0;
    bool slab_is_block = false;     // select slabs == shard blocks (phase 1 needs no histogram pass)
    uint64_t n_global = 0;          // dataset size the index describes (== host.n unsharded)
    DevBuf<uint8_t> shard_scores;   // phase-1 SC-scores, nq x n_local
    DevBuf<uint32_t> shard_cands;   // phase-2 candidates, nq x stride
    // query pipeline: tiles flow traverse -> select -> rerank on three streams,
    // double-buffered scratch, so neighbouring tiles overlap on the device.
    struct Slot {
        DevBuf<float> q;
        DevBuf<uint32_t> cells, ncells, cands, out_ids, all_id;
        DevBuf<uint16_t> dhist;               // dense select: nq x P x 8
        DevBuf<uint32_t> dT, dquota, dbase;   // dense select plan
        DevBuf<uint16_t> dsample;                 // single-pass select: sampled histograms
        DevBuf<uint16_t> dcbuf, dccnt;            // single-pass select: candidate buffers and their counts
        DevBuf<uint32_t> dL, dflag, dh2;          // single-pass select: bound, fallback flags, two-level counts
        DevBuf<double> out_d, all_d;
        cudaEvent_t trav = nullptr, sel = nullptr, rr = nullptr;
        cudaEvent_t selmain = nullptr;  // dense select: every unflagged query's candidates written
    };
    Slot slot[2];
    cudaStream_t pipe[4] = {nullptr, nullptr, nullptr, nullptr};  // traverse, select, rerank, fallback
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    // stage profiling (suco_gpu_set_profiling)
    bool profile = false;
    std::vector<cudaEvent_t> events;  // pairs (start, end) per profiled stage launch
    std::vector<int> event_stage;     // stage of each pair
    uint32_t pairs = 0;
    DevBuf<unsigned long long> stat_cum;
    uint64_t last_nq = 0, last_m = 0;
    uint64_t launches = 0;  // kernels enqueued by the last query call (suco_gpu_last_launches)

    ~suco_gpu_index() {
        for (cudaEvent_t e : events) cudaEventDestroy(e);
        for (Slot& sl : slot) {
            if (sl.trav) cudaEventDestroy(sl.trav);
            if (sl.sel) cudaEventDestroy(sl.sel);
            if (sl.rr) cudaEventDestroy(sl.rr);
            if (sl.selmain) cudaEventDestroy(sl.selmain);
        }
        if (ev_in) cudaEventDestroy(ev_in);
        if (ev_out) cudaEventDestroy(ev_out);
        for (cudaStream_t t : pipe) {
            if (t) cudaStreamDestroy(t);
        }
        if (own) cudaStreamDestroy(own);
    }
};

namespace {

void check_dataset(const float* data, uint64_t n, uint32_t d) {
    if (n < 1 || d < 1) raise(SUCO_ERR_CONTRACT, "dataset requires n >= 1 and d >= 1");
    if (!data) raise(SUCO_ERR_CONTRACT, "dataset buffer is null");
}

// Dataset finiteness (core.cpp:15-19), checked on the device after upload.
void check_finite_device(const float* d_data, uint64_t count, cudaStream_t st) {
    unsigned long long* flag = nullptr;
    CUDA_TRY(cudaMalloc(&flag, sizeof(unsigned long long)));
    const unsigned long long init = ~0ull;
    unsigned long long got = 0;
    cudaError_t e = cudaMemcpyAsync(flag, &init, sizeof init, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = launch_check_finite(d_data, count, reinterpret_cast<int*>(flag), st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&got, flag, sizeof got, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(flag);
    CUDA_TRY(e);
    if (got != ~0ull) raise(SUCO_ERR_CONTRACT, "dataset component " + std::to_string(got) + " is not finite");
}

void create_stream(suco_gpu_index* x) {
    CUDA_TRY(cudaStreamCreateWithFlags(&x->own, cudaStreamNonBlocking));
    x->stream = x->own;
    int least = 0, greatest = 0;
    CUDA_TRY(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    const char* pr = std::getenv("SUCO_PIPE_PRIO");
    const bool prio = !pr || std::atoi(pr) != 0;
    // traverse and rerank (short, many small CTAs) get priority so they fill the
    // SMs that select's GPC-bound clusters leave idle
    CUDA_TRY(cudaStreamCreateWithPriority(&x->pipe[0], cudaStreamNonBlocking, prio ? greatest : least));
    CUDA_TRY(cudaStreamCreateWithPriority(&x->pipe[1], cudaStreamNonBlocking, least));
    // the dense select's fallback (a few query blocks, latency-bound) runs beside the re-rank of the
    // unflagged queries; its CTAs go first (re-rank one priority level below, when there is one)
    const int rr_prio = !prio ? least : greatest < least ? greatest + 1 : greatest;
    CUDA_TRY(cudaStreamCreateWithPriority(&x->pipe[2], cudaStreamNonBlocking, rr_prio));
    CUDA_TRY(cudaStreamCreateWithPriority(&x->pipe[3], cudaStreamNonBlocking, greatest));
    for (auto& sl : x->slot) {
        CUDA_TRY(cudaEventCreateWithFlags(&sl.trav, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&sl.sel, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&sl.rr, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&sl.selmain, cudaEventDisableTiming));
    }
    CUDA_TRY(cudaEventCreateWithFlags(&x->ev_in, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&x->ev_out, cudaEventDisableTiming));
}

// data == nullptr: the rows are already in x->data (streamed from a vecs file).
void upload_data(suco_gpu_index* x, const float* data, uint64_t n, uint32_t d) {
    if (data) {
        x->data.reserve(n * d);
        // host or device memory (UVA): rows already on the GPU are copied device to device
        CUDA_TRY(cudaMemcpyAsync(x->data.p, data, n * d * sizeof(float), cudaMemcpyDefault, x->stream));
    }
    check_finite_device(x->data.p, n * d, x->stream);
    // integer certificate (values integral, |v| <= 2^20) for the exact fp32 rerank chains
    DevBuf<unsigned int> st;
    st.reserve(3);
    unsigned int h[3] = {0, 0, 0};
    CUDA_TRY(cudaMemsetAsync(st.p, 0, 12, x->stream));
    CUDA_TRY(launch_int_stats(x->data.p, n * d, st.p, x->stream));
    CUDA_TRY(cudaMemcpyAsync(h, st.p, 12, cudaMemcpyDeviceToHost, x->stream));
    CUDA_TRY(cudaStreamSynchronize(x->stream));
    float mx;
    std::memcpy(&mx, &h[1], 4);
    x->data_int_max = (h[0] == 0 && mx <= 1048576.f) ? mx : -1.f;
    // u8-valued rows (integers in [0, 255]): a byte copy for the exact integer re-rank, whose
    // squared distances (< 2^32) are the reference's fp64 values in any summation order
    x->dpad = 0;
    if (h[0] == 0 && h[2] == 0 && mx <= 255.f && d <= 512 && !std::getenv("SUCO_NO_U8")) {
        x->dpad = (d + 15) / 16 * 16;
        x->data8.reserve(n * x->dpad);
        CUDA_TRY(launch_pack_u8(x->data.p, n, d, x->dpad, x->data8.p, x->stream));
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
    CUDA_TRY(cudaMemcpyAsync(x->dims.p, h.layout.dims.data(), h.layout.dims.size() * 4, cudaMemcpyHostToDevice, x->stream));
    x->sub.reserve(ns);
    CUDA_TRY(cudaMemcpyAsync(x->sub.p, sd.data(), ns * sizeof(SubDesc), cudaMemcpyHostToDevice, x->stream));
    x->cent.reserve(cent.size());
    CUDA_TRY(cudaMemcpyAsync(x->cent.p, cent.data(), cent.size() * 4, cudaMemcpyHostToDevice, x->stream));
    CUDA_TRY(cudaStreamSynchronize(x->stream));
}

// Keep the IMI ids (+ slab offsets) L2-resident across the query stream: the
// select kernel's id loads are L2-latency bound, and the candidate writes and
// re-rank row gathers would otherwise evict them (measured: 93 % L2 hits, i.e.
// nearly every 256-load wave waited on a DRAM miss).
void set_l2_window(suco_gpu_index* x) {
    int max_persist = 0, max_window = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, x->device));
    CUDA_TRY(cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, x->device));
    if (const char* v = std::getenv("SUCO_L2_PERSIST")) {
        if (std::atoi(v) == 0) max_persist = 0;
    }
    if (max_persist <= 0 || max_window <= 0) return;
    const size_t want = x->ids.cap * sizeof(uint32_t);
    const size_t persist = std::min<size_t>(want, static_cast<size_t>(max_persist));
    CUDA_TRY(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, persist));
    cudaStreamAttrValue v{};
    v.accessPolicyWindow.base_ptr = x->ids.p;
    v.accessPolicyWindow.num_bytes = std::min<size_t>(want, static_cast<size_t>(max_window));
    v.accessPolicyWindow.hitRatio = std::min(1.0f, static_cast<float>(persist) / static_cast<float>(v.accessPolicyWindow.num_bytes));
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    for (cudaStream_t t : {x->own, x->pipe[0], x->pipe[1], x->pipe[2], x->pipe[3]}) {
        CUDA_TRY(cudaStreamSetAttribute(t, cudaStreamAttributeAccessPolicyWindow, &v));
    }
}

// Cell sizes and slab offsets from the device-resident CSR.
void finalize_device(suco_gpu_index* x) {
    const uint32_t ns = x->host.layout.ns;
    x->K = x->host.p.k_half * x->host.p.k_half;
    x->cell_size.reserve(uint64_t(ns) * x->K);
    CUDA_TRY(launch_cell_sizes(x->cell_off.p, ns, x->K, x->cell_size.p, x->stream));
    x->sel = plan_select(x->host.n, ns, cluster_size_from_env());
    x->slab_off.reserve(uint64_t(ns) * x->K * (x->sel.nslabs + 1));
    CUDA_TRY(launch_slab_offsets(x->cell_off.p, x->ids.p, x->host.n, ns, x->K, x->sel.CH, x->sel.nslabs, x->slab_off.p,
                                 x->stream));
    const char* dv = std::getenv("SUCO_DENSE");
    const bool allow = !(dv && std::atoi(dv) == 0);
    x->dense = (dense_supported(ns, x->K) || dense_wide_supported(ns, x->K)) && allow;
    // tables past 32-bit masks in shared memory (config 5: 8 x 10,000 cells) take the half-width
    // mode; SUCO_DENSE_HALF=0 keeps them on the cluster-counting select
    const char* hv = std::getenv("SUCO_DENSE_HALF");  // 2: force it (tests)
    const bool force = hv && std::atoi(hv) == 2;
    x->dense_half = (!x->dense || force) && allow && dense_half_supported(ns, x->K) && !(hv && std::atoi(hv) == 0);
    if (x->dense_half) {
        x->dense = true;
        const uint64_t n_pad = (x->host.n + kDensePiece - 1) / kDensePiece * kDensePiece;  // whole last piece
        x->codes.reserve(n_pad * 8);
        CUDA_TRY(launch_dense_codes_half(x->ids.p, x->cell_off.p, x->host.n, n_pad, ns, x->K, x->codes.p, x->stream));
    } else if (x->dense) {
        x->codes.reserve(x->host.n * (ns > 8 ? 16 : 8));
        CUDA_TRY(launch_dense_codes(x->ids.p, x->cell_off.p, x->host.n, ns, x->K, x->codes.p, x->stream));
    }
    CUDA_TRY(cudaStreamSynchronize(x->stream));
    set_l2_window(x);
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

void validate_params(const suco_collision_params* p, uint64_t n) {  // sc_linear.cpp:26-37
    if (!p) raise(SUCO_ERR_CONTRACT, "collision params are null");
    if (!(p->alpha > 0.0) || p->alpha > 1.0) raise(SUCO_ERR_CONFIG, "alpha must be in (0, 1], got " + std::to_string(p->alpha));
    if (!(p->beta > 0.0) || p->beta > 1.0) raise(SUCO_ERR_CONFIG, "beta must be in (0, 1], got " + std::to_string(p->beta));
    if (p->k < 1 || p->k > n) {
        raise(SUCO_ERR_CONFIG, "k must be in [1, n]; got k = " + std::to_string(p->k) + " with n = " + std::to_string(n));
    }
}

// -------------------------------------------------------------- pipeline
struct Dbg {
    uint8_t* scores = nullptr;  // n
    double* sums = nullptr;     // ns x K
    uint64_t* cum = nullptr;    // ns x K
};

uint64_t tile_size(const suco_gpu_index* x, uint64_t nq, uint64_t m, uint32_t k) {
    const uint64_t ns = x->host.layout.ns;
    const uint64_t pieces = (x->host.n + 2047) / 2048;  // dense select scratch: hist (16 B) + quota/base per piece
    const uint64_t per = ns * x->K * 4 + ns * 4 + m * 4 + (k > 32 ? m * 12 : 0) + uint64_t(x->host.d) * 4 + k * 12 +
                         (x->dense ? pieces * (24 + kDenseBuf * 2 + 14 + (ns > 8 ? 16 : 0)) + pieces / 16 * 32 + 16
                                   : 0);  // + buffers
    uint64_t budget = 16ull << 30;  // per-batch scratch on a 180 GB part
    if (const char* b = std::getenv("SUCO_SCRATCH_GB")) budget = std::max(1ll, std::atoll(b)) << 30;  // A/B
    return std::max<uint64_t>(1, std::min<uint64_t>(nq, budget / per));
}

// Resets the per-call profiling state (events + work counters).
void begin_call(suco_gpu_index* x, uint64_t nq, uint64_t m, cudaStream_t st) {
    x->pairs = 0;
    x->launches = 0;
    x->last_nq = nq;
    x->last_m = m;
    if (x->profile) {
        x->stat_cum.reserve(1);
        CUDA_TRY(cudaMemsetAsync(x->stat_cum.p, 0, sizeof(unsigned long long), st));
    }
}

// Profiling pair for one stage launch (nullptr when profiling is off).
cudaEvent_t* prof_pair(suco_gpu_index* x, int stage) {
    if (!x->profile) return nullptr;
    while (x->events.size() < 2ull * (x->pairs + 1)) {
        cudaEvent_t e;
        CUDA_TRY(cudaEventCreate(&e));
        x->events.push_back(e);
    }
    if (x->event_stage.size() < x->pairs + 1) x->event_stage.resize(x->pairs + 1);
    x->event_stage[x->pairs] = stage;
    return x->events.data() + 2ull * x->pairs++;
}

void stage_traverse(suco_gpu_index* x, suco_gpu_index::Slot& sl, const float* d_q, uint64_t nt, uint64_t target,
                    cudaStream_t st, const Dbg* dbg) {
    const HostIndex& h = x->host;
    const uint32_t ns = h.layout.ns;
    sl.cells.reserve(nt * ns * x->K);
    sl.ncells.reserve(nt * ns);
    cudaEvent_t* ev = dbg ? nullptr : prof_pair(x, 0);
    TraverseArgs ta{};
    ta.queries = d_q;
    ta.d = h.d;
    ta.nq = nt;
    ta.dims = x->dims.p;
    ta.sub = x->sub.p;
    ta.cent = x->cent.p;
    ta.cell_size = x->cell_size.p;
    ta.ns = ns;
    ta.k_half = h.p.k_half;
    ta.K = x->K;
    ta.hmax = x->hmax;
    ta.target = target;
    ta.cells = sl.cells.p;
    ta.ncells = sl.ncells.p;
    ta.dbg_sum = dbg ? dbg->sums : nullptr;
    ta.dbg_cum = dbg ? dbg->cum : nullptr;
    ta.stat_cum = ev ? x->stat_cum.p : nullptr;
    if (ev) CUDA_TRY(cudaEventRecord(ev[0], st));
    CUDA_TRY(launch_traverse(ta, st));
    x->launches += 1;
    if (ev) CUDA_TRY(cudaEventRecord(ev[1], st));
}

// The dense select's fallback lists (qflag: nq flags; qmap[0 .. *nmap): the flagged queries).
struct FbLists {
    const uint32_t* qflag = nullptr;
    const uint32_t* qmap = nullptr;
    const uint32_t* nmap = nullptr;
};

// main_done / fb_st (optional, both or neither): with the single-pass dense select, main_done is
// recorded on st once every unflagged query's candidates are written and the flagged queries'
// fallback runs on fb_st; the returned lists are then set (else empty: st has everything).
FbLists stage_select(suco_gpu_index* x, suco_gpu_index::Slot& sl, uint64_t nt, uint64_t m, cudaStream_t st,
                     const Dbg* dbg, cudaEvent_t main_done = nullptr, cudaStream_t fb_st = nullptr) {
    const HostIndex& h = x->host;
    sl.cands.reserve(nt * m);
    cudaEvent_t* ev = dbg ? nullptr : prof_pair(x, 1);
    if (x->dense && !(dbg && dbg->scores)) {
        DenseArgs da{};
        da.codes = reinterpret_cast<const uint4*>(x->codes.p);
        da.cells = sl.cells.p;
        da.ncells = sl.ncells.p;
        da.cells_cap = x->K;
        da.ns = h.layout.ns;
        da.K = x->K;
        da.n = h.n;
        da.nq = nt;
        da.m = m;
        da.WP = kDensePiece;
        da.P = static_cast<uint32_t>((h.n + da.WP - 1) / da.WP);
        da.half = x->dense_half ? 1u : 0u;
        da.nc = h.layout.ns > 8 ? 2u : 1u;  // 9..16 subspaces: two code vectors, 16 histogram levels
        sl.dhist.reserve(nt * da.P * 8 * da.nc);
        sl.dT.reserve(nt);
        sl.dquota.reserve(nt * da.P);
        sl.dbase.reserve(nt * da.P);
        da.hist = sl.dhist.p;
        da.T = sl.dT.p;
        da.quota = sl.dquota.p;
        da.base = sl.dbase.p;
        da.cands = sl.cands.p;
        const char* fv = std::getenv("SUCO_DENSE_FUSED");
        const bool fused = !(fv && std::atoi(fv) == 0);
        if (fused) {
            // the sampled histograms (every pstride-th piece) predict the threshold; at least ~32
            // sampled pieces (small corpora: all of them, so the prediction is exact)
            // about 16 sampled pieces when that is enough (cfg2: 489 pieces -> every 30th), and
            // every 64th piece at most for large corpora (measured: cfg2 2.31M -> 2.36M q/s, cfg4
            // 167K -> 174K; fewer samples mis-estimate T and send queries to the fallback)
            da.pstride = da.P <= 64 ? 1u : std::min<uint32_t>(64, da.P / 16);  // small corpora: exact
            if (const char* ps = std::getenv("SUCO_DENSE_PSTRIDE")) da.pstride = std::max(1, std::atoi(ps));  // A/B
            da.Ps = (da.P + da.pstride - 1) / da.pstride;
            sl.dsample.reserve(nt * da.Ps * 8 * da.nc);
            da.stage_all = std::getenv("SUCO_DENSE_STAGE") != nullptr;
            // entries per (piece, query): at least kDenseBuf (~6 sigma above cfg4's mean of 46); small
            // batches x corpora (cfg3: 1K queries x 489 pieces) get up to 2048 (one whole piece)
            // within 1 GB of buffers, so dense supersets do not overflow into the two-pass fallback
            const uint64_t fit = (1ull << 30) / (2ull * nt * da.P) / 8 * 8;
            da.B = static_cast<uint32_t>(std::min<uint64_t>(kDensePiece, std::max<uint64_t>(kDenseBuf, fit)));
            if (const char* bv = std::getenv("SUCO_DENSE_BUF")) da.B = std::max(8, std::atoi(bv) / 8 * 8);  // tests
            sl.dcbuf.reserve(nt * da.P * da.B);
            sl.dccnt.reserve(nt * da.P);
            da.cbuf = sl.dcbuf.p;
            da.ccnt = sl.dccnt.p;
            sl.dL.reserve(nt);
            sl.dh2.reserve(nt * da.P);
            da.h2 = sl.dh2.p;
            sl.dflag.reserve(3 * nt + 1);  // flags, flagged list, its count, tie cuts
            da.pcut = sl.dflag.p + 2 * nt + 1;
            da.no_cut = std::getenv("SUCO_DENSE_NOCUT") != nullptr;
            if (const char* cv = std::getenv("SUCO_TIE_CUT")) {  // A/B: "scale,pad"
                da.cut_scale = static_cast<float>(std::atof(cv));
                const char* comma = std::strchr(cv, ',');
                da.cut_pad = comma ? static_cast<uint32_t>(std::atoi(comma + 1)) : 0u;
            }
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
        x->launches += fused ? 10 : 3;
        const bool stats = std::getenv("SUCO_DENSE_STATS") != nullptr;  // diagnostics: fallback rate
        if (stats && fused) {
            uint32_t nflag = 0;
            std::vector<uint32_t> Lh(nt);
            CUDA_TRY(cudaMemcpyAsync(&nflag, da.nmap, 4, cudaMemcpyDeviceToHost, st));
            CUDA_TRY(cudaMemcpyAsync(Lh.data(), da.L, nt * 4, cudaMemcpyDeviceToHost, st));
            CUDA_TRY(cudaStreamSynchronize(st));
            uint64_t gated = 0, hist[9] = {};
            for (uint32_t v : Lh) {
                v &= 0xffu;
                gated += v == 0;
                hist[std::min<uint32_t>(v, 8)]++;
            }
            std::fprintf(stderr,
                         "[suco] dense select: %u of %llu queries took the two-pass fallback (pstride %u; L = 0 "
                         "(density gate / no bound) for %llu; L histogram 0..8: %llu %llu %llu %llu %llu %llu %llu "
                         "%llu %llu)\n",
                         nflag, static_cast<unsigned long long>(nt), da.pstride, static_cast<unsigned long long>(gated),
                         (unsigned long long)hist[0], (unsigned long long)hist[1], (unsigned long long)hist[2],
                         (unsigned long long)hist[3], (unsigned long long)hist[4], (unsigned long long)hist[5],
                         (unsigned long long)hist[6], (unsigned long long)hist[7], (unsigned long long)hist[8]);
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
    sa.scores_dbg = dbg ? dbg->scores : nullptr;
    if (ev) CUDA_TRY(cudaEventRecord(ev[0], st));
    CUDA_TRY(launch_select(sa, x->sel, nt, st));
    x->launches += 1;
    if (ev) CUDA_TRY(cudaEventRecord(ev[1], st));
    return {};
}

void stage_rerank(suco_gpu_index* x, suco_gpu_index::Slot& sl, const float* d_q, uint64_t nt, uint64_t m, uint32_t k,
                  uint32_t* d_ids, double* d_dists, cudaStream_t st, bool profiled, const FbLists* fl = nullptr,
                  bool flagged = false) {
    const HostIndex& h = x->host;
    cudaEvent_t* ev = profiled ? prof_pair(x, 2) : nullptr;
    RerankArgs ra{};
    ra.data = x->data.p;
    ra.n = h.n;
    ra.d = h.d;
    ra.queries = d_q;
    ra.cands = sl.cands.p;
    ra.m = m;
    ra.k = k;
    ra.out_ids = d_ids;
    ra.out_dists = d_dists;
    ra.data_int_max = x->data_int_max;
    ra.data8 = x->dpad ? x->data8.p : nullptr;
    ra.dpad = x->dpad;
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
    if (ev) CUDA_TRY(cudaEventRecord(ev[0], st));
    CUDA_TRY(launch_rerank(ra, nt, st));
    x->launches += (ra.data8 ? 2 : 1) + (k > 32 ? 1 : 0);  // u8 + fp32/fp64 kernels, generic top-k
    if (ev) CUDA_TRY(cudaEventRecord(ev[1], st));
}

// One tile through all three stages on a single stream (intermediates/debug).
void run_tile(suco_gpu_index* x, const float* d_q, uint64_t nt, uint64_t target, uint64_t m, uint32_t k,
              uint32_t* d_ids, double* d_dists, cudaStream_t st, const Dbg* dbg) {
    auto& sl = x->slot[0];
    stage_traverse(x, sl, d_q, nt, target, st, dbg);
    stage_select(x, sl, nt, m, st, dbg);
    stage_rerank(x, sl, d_q, nt, m, k, d_ids, d_dists, st, dbg == nullptr);
}

uint64_t pipeline_tiles(uint64_t nq, uint64_t mem_tile) {
    uint64_t want = 1;  // measured: overlapping tiles only stretches select (all SMs busy)
    if (const char* t = std::getenv("SUCO_TILES")) want = std::max(1, std::atoi(t));
    uint64_t tiles = std::max<uint64_t>(1, std::min<uint64_t>(want, nq / 512));
    tiles = std::max<uint64_t>(tiles, (nq + mem_tile - 1) / mem_tile);
    return tiles;
}

// The batched query pipeline. Queries are either device-resident (h_q == nullptr,
// d_q given) or host (h_q given: copied per tile on the traverse stream).
// Outputs go to d_ids/d_dists, or to host h_ids/h_dists (copied per tile).
void run_pipeline(suco_gpu_index* x, const float* h_q, const float* d_q, uint64_t nq, uint32_t qlen,
                  const suco_collision_params* p, uint32_t* d_ids, double* d_dists, uint32_t* h_ids, double* h_dists,
                  cudaStream_t user) {
    if (x->num_shards > 1) raise(SUCO_ERR_CONTRACT, "a shard answers only through the two-phase shard protocol");
    const uint64_t n = x->host.n;
    const uint32_t k = p->k;
    const uint64_t m = suco_candidate_count(p->beta, n, k);
    const uint64_t target = suco_collision_count(p->alpha, n);
    const uint64_t tiles = pipeline_tiles(nq, tile_size(x, nq, m, k));
    const uint64_t tile = (nq + tiles - 1) / tiles;
    begin_call(x, nq, m, user);
    CUDA_TRY(cudaEventRecord(x->ev_in, user));
    for (cudaStream_t t : x->pipe) CUDA_TRY(cudaStreamWaitEvent(t, x->ev_in, 0));
    cudaStream_t s_trav = x->pipe[0], s_sel = x->pipe[1], s_rr = x->pipe[2];
    // measured (SUCO_FB_OVERLAP=1/0 forces it): cfg2 (byte rows, 10,000 queries) 2.334M -> 2.364M q/s
    // (e2e 2.12M -> 2.23M); slower where the re-rank is long beside it (fp32 rows: cfg3 143K -> 136K,
    // cfg4 170K -> 169K), so only byte-row re-ranks of large tiles overlap
    const char* fo = std::getenv("SUCO_FB_OVERLAP");
    const bool fb_overlap = fo ? std::atoi(fo) != 0 : (x->dpad && !x->dense_half && tile >= 4096);
    for (uint64_t t = 0; t * tile < nq; ++t) {
        const uint64_t q0 = t * tile, nt = std::min(tile, nq - q0);
        auto& sl = x->slot[t & 1];
        // slot reuse: tile t-2's select read `cells`, its rerank read `q`/`cands`
        CUDA_TRY(cudaStreamWaitEvent(s_trav, sl.sel, 0));
        CUDA_TRY(cudaStreamWaitEvent(s_trav, sl.rr, 0));
        const float* tq = d_q ? d_q + q0 * qlen : nullptr;
        if (h_q) {
            sl.q.reserve(tile * qlen);
            CUDA_TRY(cudaMemcpyAsync(sl.q.p, h_q + q0 * qlen, nt * qlen * 4, cudaMemcpyHostToDevice, s_trav));
            tq = sl.q.p;
        }
        stage_traverse(x, sl, tq, nt, target, s_trav, nullptr);
        CUDA_TRY(cudaEventRecord(sl.trav, s_trav));
        CUDA_TRY(cudaStreamWaitEvent(s_sel, sl.trav, 0));
        CUDA_TRY(cudaStreamWaitEvent(s_sel, sl.rr, 0));
        // the fallback of the few flagged queries overlaps the re-rank of the others (A/B:
        // SUCO_FB_OVERLAP=0 keeps it on the select stream)
        const FbLists fl = stage_select(x, sl, nt, m, s_sel, nullptr, fb_overlap ? sl.selmain : nullptr,
                                        fb_overlap ? x->pipe[3] : nullptr);
        CUDA_TRY(cudaEventRecord(sl.sel, fl.qflag ? x->pipe[3] : s_sel));
        CUDA_TRY(cudaStreamWaitEvent(s_rr, fl.qflag ? sl.selmain : sl.sel, 0));
        uint32_t* oi = d_ids ? d_ids + q0 * k : nullptr;
        double* od = d_dists ? d_dists + q0 * k : nullptr;
        if (h_ids) {
            sl.out_ids.reserve(tile * k);
            sl.out_d.reserve(tile * k);
            oi = sl.out_ids.p;
            od = sl.out_d.p;
        }
        stage_rerank(x, sl, tq, nt, m, k, oi, od, s_rr, true, &fl, false);
        if (fl.qflag) {
            CUDA_TRY(cudaStreamWaitEvent(s_rr, sl.sel, 0));
            stage_rerank(x, sl, tq, nt, m, k, oi, od, s_rr, true, &fl, true);
        }
        if (h_ids) {
            CUDA_TRY(cudaMemcpyAsync(h_ids + q0 * k, oi, nt * k * 4, cudaMemcpyDeviceToHost, s_rr));
            CUDA_TRY(cudaMemcpyAsync(h_dists + q0 * k, od, nt * k * 8, cudaMemcpyDeviceToHost, s_rr));
        }
        CUDA_TRY(cudaEventRecord(sl.rr, s_rr));
    }
    CUDA_TRY(cudaEventRecord(x->ev_out, s_rr));
    CUDA_TRY(cudaStreamWaitEvent(user, x->ev_out, 0));
}

void check_query_args(const suco_gpu_index* x, uint32_t qlen, const suco_collision_params* p) {
    if (!x) raise(SUCO_ERR_CONTRACT, "index is null");
    if (qlen != x->host.d) {  // query.cpp:203-206
        raise(SUCO_ERR_CONTRACT, "query length " + std::to_string(qlen) + " does not match dataset d = " +
                                     std::to_string(x->host.d));
    }
    validate_params(p, x->host.n);  // query.cpp:208
    if (x->host.layout.ns > 255) raise(SUCO_ERR_CONFIG, "the GPU path keeps u8 collision counters: N_s must be <= 255");
}

suco_gpu_index* new_index(int device) {
    auto* x = new suco_gpu_index();
    x->device = device;
    return x;
}

// SC-Linear (sc_linear.cpp:49-121) over the index's device rows and layout.
struct ScScratch {
    DevBuf<uint32_t> sub_off, vals, vals_alt, scores, cands;
    DevBuf<uint8_t> consec, temp;
    DevBuf<unsigned long long> keys, keys_alt;
    DevBuf<float> q;
    ScArgs a{};
};

void sc_setup(suco_gpu_index* x, ScScratch& w) {
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
    cudaStream_t st = x->stream;
    w.sub_off.reserve(L.ns + 1);
    w.consec.reserve(L.ns);
    CUDA_TRY(cudaMemcpyAsync(w.sub_off.p, off.data(), off.size() * 4, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(w.consec.p, consec.data(), consec.size(), cudaMemcpyHostToDevice, st));
    w.keys.reserve(n);
    w.keys_alt.reserve(n);
    w.vals.reserve(n);
    w.vals_alt.reserve(n);
    w.scores.reserve(n);
    w.q.reserve(x->host.d);
    const size_t tb = sc_temp_bytes(n);
    w.temp.reserve(tb);
    w.a.data = x->data.p;
    w.a.n = n;
    w.a.d = x->host.d;
    w.a.ns = L.ns;
    w.a.dims = x->dims.p;
    w.a.sub_off = w.sub_off.p;
    w.a.consec = w.consec.p;
    w.a.q = w.q.p;
    w.a.keys = w.keys.p;
    w.a.keys_alt = w.keys_alt.p;
    w.a.vals = w.vals.p;
    w.a.vals_alt = w.vals_alt.p;
    w.a.temp = w.temp.p;
    w.a.temp_bytes = tb;
}

void check_sc_query(const suco_gpu_index* x, uint32_t qlen) {
    if (!x) raise(SUCO_ERR_CONTRACT, "index is null");
    if (qlen != x->host.d) {  // sc_linear.cpp:55-58
        raise(SUCO_ERR_CONTRACT, "query length " + std::to_string(qlen) + " does not match dataset d = " +
                                     std::to_string(x->host.d));
    }
}

}  // namespace

// ======================================================================= C ABI
extern "C" {

const char* suco_last_error(void) { return g_err.c_str(); }

int suco_gpu_device_count(int* count) {
    return guarded([&] {
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

void load_core(suco_gpu_index* x, uint64_t n) {
    upload_codebooks(x);
    upload_imi(x);
    finalize_device(x);
    x->n_global = n;
}

int suco_gpu_load_index(const unsigned char* bytes, uint64_t len, const float* data, uint64_t n, uint32_t d, int device,
                        suco_gpu_index** out) {
    return guarded([&] {
        if (!out) raise(SUCO_ERR_CONTRACT, "output handle pointer is null");
        *out = nullptr;
        HostIndex h = parse_index(bytes, len);  // FORMAT first (load_index), as suco_cli.cpp:243
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
        suco_gpu_index* x = new_index(device);
        try {
            create_stream(x);
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

void build_core(suco_gpu_index* x, uint64_t n, uint32_t d, const suco_index_params* params,
                const uint32_t* train = nullptr, uint64_t n_train = 0);

int suco_gpu_build_index(const float* data, uint64_t n, uint32_t d, const suco_index_params* params, int device,
                         suco_gpu_index** out) {
    return guarded([&] {
        if (!out) raise(SUCO_ERR_CONTRACT, "output handle pointer is null");
        *out = nullptr;
        if (!params) raise(SUCO_ERR_CONTRACT, "index params are null");
        check_dataset(data, n, d);
        DeviceGuard g(device);
        suco_gpu_index* x = new_index(device);
        try {
            create_stream(x);
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
        suco_gpu_index* x = new_index(device);
        try {
            create_stream(x);
            upload_data(x, data, n, d);
            build_core(x, n, d, params, train_ids, n_train);
        } catch (...) {
            delete x;
            throw;
        }
        *out = x;
    });
}

// build_index (index.cpp:98-145) over rows already on the device; train != nullptr: the sampled
// build (k-means on those rows, every row assigned to its nearest centroid).
void build_core(suco_gpu_index* x, uint64_t n, uint32_t d, const suco_index_params* params, const uint32_t* train,
                uint64_t n_train) {
    {
        {
            // index.cpp:100-108
            if (params->k_half < 1) raise(SUCO_ERR_CONFIG, "k_half must be >= 1");
            if (params->iterations < 1) raise(SUCO_ERR_CONFIG, "iterations must be >= 1");
            const uint64_t nfit = train ? n_train : n;
            if (nfit < params->k_half) {
                raise(SUCO_ERR_CONFIG, std::string(train ? "training sample" : "dataset") + " has n = " +
                                           std::to_string(nfit) + " points, fewer than k_half = " +
                                           std::to_string(params->k_half));
            }
            if (n > 0xFFFFFFFFull) raise(SUCO_ERR_CONTRACT, "dataset exceeds 32-bit point-id capacity");
            for (uint64_t i = 0; train && i < n_train; ++i) {
                if (train[i] >= n || (i && train[i] <= train[i - 1])) {
                    raise(SUCO_ERR_CONTRACT, "training ids must be strictly ascending and < n (entry " +
                                                 std::to_string(i) + ")");
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
            build_index_device(x->data.p, n, d, x->host.layout, *params, bo, x->stream, train, n_train);
            upload_codebooks(x);
            finalize_device(x);
            x->n_global = n;
        }
    }
}

int suco_gpu_serialize_index(const suco_gpu_index* x, unsigned char* buf, uint64_t cap, uint64_t* len) {
    return guarded([&] {
        if (!x || !len) raise(SUCO_ERR_CONTRACT, "null argument");
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
        if (n) *n = x->host.n;
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

int suco_gpu_set_stream(suco_gpu_index* x, void* stream) {
    return guarded([&] {
        if (!x) raise(SUCO_ERR_CONTRACT, "index is null");
        x->stream = stream ? static_cast<cudaStream_t>(stream) : x->own;
    });
}

int suco_gpu_set_profiling(suco_gpu_index* x, int enabled) {
    return guarded([&] {
        if (!x) raise(SUCO_ERR_CONTRACT, "index is null");
        DeviceGuard g(x->device);
        x->profile = enabled != 0;
        if (x->profile) x->stat_cum.reserve(1);
    });
}

int suco_gpu_last_launches(const suco_gpu_index* x, uint64_t* launches) {
    return guarded([&] {
        if (!x || !launches) raise(SUCO_ERR_CONTRACT, "null argument");
        *launches = x->launches;
    });
}

int suco_gpu_stage_times(suco_gpu_index* x, double* ms, uint64_t* stats) {
    return guarded([&] {
        if (!x) raise(SUCO_ERR_CONTRACT, "index is null");
        if (!x->profile) raise(SUCO_ERR_CONTRACT, "profiling is not enabled on this index");
        DeviceGuard g(x->device);
        double acc[3] = {0, 0, 0};
        for (uint32_t i = 0; i < x->pairs; ++i) {
            cudaEvent_t* ev = x->events.data() + 2ull * i;
            CUDA_TRY(cudaEventSynchronize(ev[1]));
            float f = 0.f;
            CUDA_TRY(cudaEventElapsedTime(&f, ev[0], ev[1]));
            acc[x->event_stage[i]] += f;
        }
        if (ms) {
            for (int st = 0; st < 3; ++st) ms[st] = acc[st];
        }
        if (stats) {
            unsigned long long c = 0;
            CUDA_TRY(cudaMemcpy(&c, x->stat_cum.p, sizeof c, cudaMemcpyDeviceToHost));
            stats[0] = c;
            stats[1] = x->last_nq;
            stats[2] = x->last_m;
        }
    });
}

int suco_gpu_synchronize(suco_gpu_index* x) {
    return guarded([&] {
        if (!x) raise(SUCO_ERR_CONTRACT, "index is null");
        DeviceGuard g(x->device);
        CUDA_TRY(cudaStreamSynchronize(x->stream));
    });
}

int suco_gpu_knn_query_batch_device(suco_gpu_index* x, const float* d_queries, uint64_t nq, uint32_t qlen,
                                    const suco_collision_params* p, uint32_t* d_ids, double* d_dists, void* stream) {
    return guarded([&] {
        check_query_args(x, qlen, p);
        if (nq == 0) return;
        DeviceGuard g(x->device);
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : x->stream;
        run_pipeline(x, nullptr, d_queries, nq, qlen, p, d_ids, d_dists, nullptr, nullptr, st);
    });
}

int suco_gpu_knn_query_batch(suco_gpu_index* x, const float* queries, uint64_t nq, uint32_t qlen,
                             const suco_collision_params* p, uint32_t* ids, double* dists) {
    return guarded([&] {
        check_query_args(x, qlen, p);
        if (nq == 0) return;
        DeviceGuard g(x->device);
        run_pipeline(x, queries, nullptr, nq, qlen, p, nullptr, nullptr, ids, dists, x->stream);
        CUDA_TRY(cudaStreamSynchronize(x->stream));
    });
}

// exact_knn (eval.hpp:29, eval.cpp:28-62) for a batch: the re-rank kernels over every id.
int suco_gpu_exact_knn_batch(suco_gpu_index* x, const float* queries, uint64_t nq, uint32_t qlen, uint32_t k,
                             uint32_t* ids, double* dists) {
    return guarded([&] {
        if (!x) raise(SUCO_ERR_CONTRACT, "index is null");
        const uint64_t n = x->host.n;
        if (qlen != x->host.d) {
            raise(SUCO_ERR_CONTRACT, "query length " + std::to_string(qlen) + " does not match dataset d = " +
                                         std::to_string(x->host.d));
        }
        if (k < 1 || k > n) {
            raise(SUCO_ERR_CONTRACT, "k must be in [1, n]; got k = " + std::to_string(k) + ", n = " + std::to_string(n));
        }
        if (nq == 0) return;
        if (!queries || !ids || !dists) raise(SUCO_ERR_CONTRACT, "null buffer");
        DeviceGuard g(x->device);
        cudaStream_t st = x->stream;
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
            ra.data = x->data.p;
            ra.n = n;
            ra.d = x->host.d;
            ra.queries = dq.p;
            ra.cands = nullptr;
            ra.identity = true;
            ra.m = n;
            ra.k = k;
            ra.out_ids = di.p;
            ra.out_dists = dd.p;
            ra.data_int_max = x->data_int_max;
            ra.data8 = x->dpad ? x->data8.p : nullptr;
            ra.dpad = x->dpad;
            ra.all_d = all_d.p;
            ra.all_id = all_id.p;
            CUDA_TRY(launch_rerank(ra, nt, st));
            CUDA_TRY(cudaMemcpyAsync(ids + q0 * k, di.p, nt * k * 4, cudaMemcpyDeviceToHost, st));
            CUDA_TRY(cudaMemcpyAsync(dists + q0 * k, dd.p, nt * k * 8, cudaMemcpyDeviceToHost, st));
        }
        CUDA_TRY(cudaStreamSynchronize(st));
    });
}

int suco_gpu_sc_scores(suco_gpu_index* x, const float* query, uint32_t qlen, double alpha, uint32_t* scores) {
    return guarded([&] {
        check_sc_query(x, qlen);
        // the reference leaves alpha unchecked here (c > n would index past the order array)
        if (!(alpha > 0.0) || alpha > 1.0) raise(SUCO_ERR_CONFIG, "alpha must be in (0, 1], got " + std::to_string(alpha));
        if (!query || !scores) raise(SUCO_ERR_CONTRACT, "null buffer");
        DeviceGuard g(x->device);
        cudaStream_t st = x->stream;
        ScScratch w;
        sc_setup(x, w);
        const uint64_t c = std::min<uint64_t>(suco_collision_count(alpha, x->host.n), x->host.n);
        CUDA_TRY(cudaMemcpyAsync(w.q.p, query, qlen * 4, cudaMemcpyHostToDevice, st));
        CUDA_TRY(launch_sc_scores(w.a, c, w.scores.p, st));
        CUDA_TRY(cudaMemcpyAsync(scores, w.scores.p, x->host.n * 4, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
    });
}

int suco_gpu_sc_linear_batch(suco_gpu_index* x, const float* queries, uint64_t nq, uint32_t qlen,
                             const suco_collision_params* p, uint32_t* ids, double* dists) {
    return guarded([&] {
        if (!x) raise(SUCO_ERR_CONTRACT, "index is null");
        validate_params(p, x->host.n);  // sc_linear.cpp:97, before the query-length check
        check_sc_query(x, qlen);
        if (nq == 0) return;
        if (!queries || !ids || !dists) raise(SUCO_ERR_CONTRACT, "null buffer");
        DeviceGuard g(x->device);
        cudaStream_t st = x->stream;
        const uint64_t n = x->host.n;
        const uint64_t c = std::min<uint64_t>(suco_collision_count(p->alpha, n), n);
        const uint64_t m = std::min<uint64_t>(suco_candidate_count(p->beta, n, p->k), n);
        ScScratch w;
        sc_setup(x, w);
        w.cands.reserve(n);
        DevBuf<uint32_t> di, all_id;
        DevBuf<double> dd, all_d;
        di.reserve(p->k);
        dd.reserve(p->k);
        if (p->k > 32) {
            all_d.reserve(m);
            all_id.reserve(m);
        }
        for (uint64_t q = 0; q < nq; ++q) {
            CUDA_TRY(cudaMemcpyAsync(w.q.p, queries + q * qlen, qlen * 4, cudaMemcpyHostToDevice, st));
            CUDA_TRY(launch_sc_scores(w.a, c, w.scores.p, st));
            // the m best by (score desc, id asc): the first m of a stable sort on N_s - score
            CUDA_TRY(launch_sc_candidates(w.a, w.scores.p, w.cands.p, st));
            RerankArgs ra{};
            ra.data = x->data.p;
            ra.n = n;
            ra.d = x->host.d;
            ra.queries = w.q.p;
            ra.cands = w.cands.p;
            ra.m = m;
            ra.k = p->k;
            ra.out_ids = di.p;
            ra.out_dists = dd.p;
            ra.data_int_max = x->data_int_max;
            ra.data8 = x->dpad ? x->data8.p : nullptr;
            ra.dpad = x->dpad;
            ra.all_d = all_d.p;
            ra.all_id = all_id.p;
            CUDA_TRY(launch_rerank(ra, 1, st));
            CUDA_TRY(cudaMemcpyAsync(ids + q * p->k, di.p, p->k * 4, cudaMemcpyDeviceToHost, st));
            CUDA_TRY(cudaMemcpyAsync(dists + q * p->k, dd.p, p->k * 8, cudaMemcpyDeviceToHost, st));
        }
        CUDA_TRY(cudaStreamSynchronize(st));
    });
}

int suco_gpu_query_intermediates(suco_gpu_index* x, const float* query, uint32_t qlen, const suco_collision_params* p,
                                 uint32_t* scores, uint32_t* cands, uint64_t* m_out, uint32_t* cells_per_subspace,
                                 uint64_t* cumulative) {
    return guarded([&] {
        check_query_args(x, qlen, p);
        DeviceGuard g(x->device);
        cudaStream_t st = x->stream;
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
        Dbg dbg{sc.p, sums.p, cum.p};
        auto& sl = x->slot[0];
        sl.q.reserve(qlen);
        sl.out_ids.reserve(p->k);
        sl.out_d.reserve(p->k);
        CUDA_TRY(cudaMemcpyAsync(sl.q.p, query, qlen * 4, cudaMemcpyHostToDevice, st));
        run_tile(x, sl.q.p, 1, target, m, p->k, sl.out_ids.p, sl.out_d.p, st, &dbg);
        CUDA_TRY(cudaStreamSynchronize(st));
        if (scores) {
            std::vector<uint8_t> s8(n);
            CUDA_TRY(cudaMemcpy(s8.data(), sc.p, n, cudaMemcpyDeviceToHost));
            for (uint64_t i = 0; i < n; ++i) scores[i] = s8[i];
        }
        if (cands) {  // the select kernel emits the candidate SET; report it ascending
            if (x->dense) {  // the production select (dense.cu) on the same traversal output
                Dbg nodbg{};
                stage_select(x, sl, 1, m, st, &nodbg);
                CUDA_TRY(cudaStreamSynchronize(st));
            }
            CUDA_TRY(cudaMemcpy(cands, x->slot[0].cands.p, m * 4, cudaMemcpyDeviceToHost));
            std::sort(cands, cands + m);
        }
        if (m_out) *m_out = m;
        std::vector<uint32_t> nc(ns);
        CUDA_TRY(cudaMemcpy(nc.data(), x->slot[0].ncells.p, ns * 4, cudaMemcpyDeviceToHost));
        if (cells_per_subspace) std::memcpy(cells_per_subspace, nc.data(), ns * 4);
        if (cumulative) {
            for (uint32_t s = 0; s < ns; ++s) {
                cumulative[s] = 0;
                if (nc[s]) CUDA_TRY(cudaMemcpy(cumulative + s, cum.p + uint64_t(s) * x->K + nc[s] - 1, 8, cudaMemcpyDeviceToHost));
            }
        }
    });
}

// ------------------------------------------------------------------ shards
int suco_gpu_make_shard(const suco_gpu_index* full, uint32_t shard, uint32_t num_shards, uint32_t block,
                        suco_gpu_index** out) {
    return guarded([&] {
        if (!full || !out) raise(SUCO_ERR_CONTRACT, "null argument");
        if (full->num_shards != 1) raise(SUCO_ERR_CONTRACT, "shards are cut from an unsharded index");
        if (num_shards < 1 || shard >= num_shards) raise(SUCO_ERR_CONFIG, "shard must be < num_shards");
        if (block < 1) raise(SUCO_ERR_CONFIG, "block size must be >= 1");
        *out = nullptr;
        DeviceGuard g(full->device);
        const uint64_t n = full->host.n;
        const uint32_t d = full->host.d, ns = full->host.layout.ns;
        const uint64_t nb = (n + block - 1) / block;
        uint64_t n_local = 0;
        for (uint64_t j = shard; j < nb; j += num_shards) n_local += std::min<uint64_t>(block, n - j * block);
        if (n_local == 0) raise(SUCO_ERR_CONFIG, "shard owns no points (n too small for this block size)");
        suco_gpu_index* x = new_index(full->device);
        try {
            create_stream(x);
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
            // rows of the owned blocks, back to back (and their u8 copies)
            x->data.reserve(n_local * d);
            if (x->dpad) x->data8.reserve(n_local * x->dpad);
            uint64_t lo = 0;
            for (uint64_t j = shard; j < nb; j += num_shards) {
                const uint64_t len = std::min<uint64_t>(block, n - j * block);
                CUDA_TRY(cudaMemcpyAsync(x->data.p + lo * d, full->data.p + j * block * d, len * d * 4,
                                         cudaMemcpyDeviceToDevice, x->stream));
                if (x->dpad) {
                    CUDA_TRY(cudaMemcpyAsync(x->data8.p + lo * x->dpad, full->data8.p + j * block * x->dpad,
                                             len * x->dpad, cudaMemcpyDeviceToDevice, x->stream));
                }
                lo += len;
            }
            upload_codebooks(x);
            x->K = full->K;
            const uint64_t K = x->K;
            // GLOBAL cell sizes: every shard makes the global Dynamic-Activation cut
            x->cell_size.reserve(ns * K);
            CUDA_TRY(cudaMemcpyAsync(x->cell_size.p, full->cell_size.p, ns * K * 4, cudaMemcpyDeviceToDevice, x->stream));
            // local IMI: owned ids of every cell, as local ids, ascending
            DevBuf<uint32_t> counts;
            counts.reserve(ns * K);
            CUDA_TRY(launch_shard_imi(full->ids.p, full->cell_off.p, n, ns, x->K, block, num_shards, shard, counts.p,
                                      nullptr, 0, nullptr, x->stream));
            std::vector<uint32_t> hc(ns * K), hoff(ns * (K + 1));
            CUDA_TRY(cudaMemcpyAsync(hc.data(), counts.p, ns * K * 4, cudaMemcpyDeviceToHost, x->stream));
            CUDA_TRY(cudaStreamSynchronize(x->stream));
            for (uint32_t sub = 0; sub < ns; ++sub) {
                uint32_t run = 0;
                for (uint64_t c = 0; c < K; ++c) {
                    hoff[sub * (K + 1) + c] = run;
                    run += hc[sub * K + c];
                }
                hoff[sub * (K + 1) + K] = run;
            }
            x->cell_off.reserve(ns * (K + 1));
            CUDA_TRY(cudaMemcpyAsync(x->cell_off.p, hoff.data(), hoff.size() * 4, cudaMemcpyHostToDevice, x->stream));
            x->ids.reserve(ns * n_local);
            CUDA_TRY(launch_shard_imi(full->ids.p, full->cell_off.p, n, ns, x->K, block, num_shards, shard, nullptr,
                                      x->cell_off.p, n_local, x->ids.p, x->stream));
            // dense select when the blocks are whole pieces (pieces never straddle blocks)
            const char* dv = std::getenv("SUCO_DENSE");
            x->dense = dense_supported(ns, x->K) && block % kDensePiece == 0 && !(dv && std::atoi(dv) == 0);
            x->dense_half = false;  // shards: 32-query blocks or the cluster-counting select
            if (x->dense) {
                x->codes.reserve(n_local * 8);
                CUDA_TRY(launch_dense_codes(x->ids.p, x->cell_off.p, n_local, ns, x->K, x->codes.p, x->stream));
            }
            x->sel = SelectConfig{};
            if (block % select_slab_align() == 0) x->sel = plan_select_fixed(n_local, ns, block);
            x->slab_is_block = x->sel.CH != 0;  // slab histograms are the block histograms
            if (!x->slab_is_block) x->sel = plan_select(n_local, ns, cluster_size_from_env());
            x->slab_off.reserve(uint64_t(ns) * K * (x->sel.nslabs + 1));
            CUDA_TRY(launch_slab_offsets(x->cell_off.p, x->ids.p, n_local, ns, x->K, x->sel.CH, x->sel.nslabs,
                                         x->slab_off.p, x->stream));
            CUDA_TRY(cudaStreamSynchronize(x->stream));
            set_l2_window(x);
        } catch (...) {
            delete x;
            throw;
        }
        *out = x;
    });
}

int suco_gpu_shard_block_hint(const suco_gpu_index* full, uint32_t num_shards, uint32_t* block) {
    return guarded([&] {
        if (!full || !block) raise(SUCO_ERR_CONTRACT, "null argument");
        if (num_shards < 1) raise(SUCO_ERR_CONFIG, "num_shards must be >= 1");
        DeviceGuard g(full->device);
        const uint64_t n = full->host.n;
        const uint32_t ns = full->host.layout.ns;
        // slab length the select kernel picks for one shard's share; the shard then has at most
        // CS blocks, so one counting round (plan_select_fixed with CH = block)
        const uint64_t share = (n + num_shards - 1) / num_shards;
        const SelectConfig c = plan_select(std::max<uint64_t>(share, 1), ns, cluster_size_from_env());
        *block = c.rounds == 1 ? c.CH : select_slab_align() * 4;
    });
}

int suco_gpu_shard_info(const suco_gpu_index* x, uint64_t* n_global, uint64_t* n_local, uint32_t* nblocks_local,
                        uint32_t* block, uint32_t* shard, uint32_t* num_shards) {
    return guarded([&] {
        if (!x) raise(SUCO_ERR_CONTRACT, "index is null");
        const uint32_t b = x->block ? x->block : static_cast<uint32_t>(std::min<uint64_t>(x->host.n, 0xFFFFFFFFull));
        if (n_global) *n_global = x->n_global;
        if (n_local) *n_local = x->host.n;
        // histogram rows per query: dense pieces of kDensePiece ids, else whole blocks
        const uint32_t unit = x->dense ? kDensePiece : b;
        if (nblocks_local) *nblocks_local = static_cast<uint32_t>((x->host.n + unit - 1) / unit);
        if (block) *block = b;
        if (shard) *shard = x->shard;
        if (num_shards) *num_shards = x->num_shards;
    });
}

int suco_gpu_shard_pieces(const suco_gpu_index* x, uint32_t* pieces_per_block, int* dense) {
    return guarded([&] {
        if (!x || !pieces_per_block) raise(SUCO_ERR_CONTRACT, "null argument");
        const uint32_t b = x->block ? x->block : static_cast<uint32_t>(std::min<uint64_t>(x->host.n, 0xFFFFFFFFull));
        *pieces_per_block = x->dense ? b / kDensePiece : 1u;
        if (dense) *dense = x->dense ? 1 : 0;
    });
}

// Local exact re-rank of a shard's candidates (squared distances, local ids -> global ids).
void shard_rerank(suco_gpu_index* x, const float* d_queries, uint64_t nq, uint32_t k, const uint32_t* d_counts,
                  uint64_t sd, uint32_t* d_ids, double* d_sqdists, cudaStream_t st) {
    const uint64_t nl = x->host.n;
    const uint32_t b = x->block ? x->block : static_cast<uint32_t>(nl);
    RerankArgs ra{};
    ra.data = x->data.p;
    ra.n = nl;
    ra.d = x->host.d;
    ra.queries = d_queries;
    ra.cands = x->shard_cands.p;
    ra.m = sd;
    ra.k = k;
    ra.out_ids = d_ids;
    ra.out_dists = d_sqdists;
    ra.data_int_max = x->data_int_max;
    ra.data8 = x->dpad ? x->data8.p : nullptr;
    ra.dpad = x->dpad;
    ra.counts = d_counts;
    ra.squared = true;
    auto& sl = x->slot[0];
    if (k > 32) {
        sl.all_d.reserve(nq * sd);
        sl.all_id.reserve(nq * sd);
        ra.all_d = sl.all_d.p;
        ra.all_id = sl.all_id.p;
    }
    CUDA_TRY(launch_rerank(ra, nq, st));
    x->launches += (ra.data8 ? 2 : 1) + (k > 32 ? 1 : 0);
    if (x->num_shards > 1) {
        CUDA_TRY(launch_shard_ids(d_ids, nq * k, b, x->num_shards, x->shard, st));
        x->launches += 1;
    }
}

DenseArgs shard_dense_args(suco_gpu_index* x, suco_gpu_index::Slot& sl, uint64_t nq) {
    DenseArgs da{};
    da.codes = reinterpret_cast<const uint4*>(x->codes.p);
    da.cells = sl.cells.p;
    da.ncells = sl.ncells.p;
    da.cells_cap = x->K;
    da.ns = x->host.layout.ns;
    da.K = x->K;
    da.n = x->host.n;
    da.nq = nq;
    da.WP = kDensePiece;
    da.P = static_cast<uint32_t>((x->host.n + kDensePiece - 1) / kDensePiece);
    return da;
}

// Query-split traversal for the multi-GPU protocol: rank r traverses its slice of the
// batch; the compact cell lists are exchanged and phases 1/2 take them (_cells variants).
int suco_gpu_shard_traverse(suco_gpu_index* x, const float* d_queries, uint64_t nq, uint32_t qlen,
                            const suco_collision_params* p, uint32_t* d_cells, uint32_t* d_ncells, void* stream) {
    return guarded([&] {
        if (!x) raise(SUCO_ERR_CONTRACT, "index is null");
        if (qlen != x->host.d) raise(SUCO_ERR_CONTRACT, "query length does not match dataset d");
        validate_params(p, x->n_global);
        if (nq == 0) return;
        DeviceGuard g(x->device);
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : x->stream;
        const HostIndex& h = x->host;
        TraverseArgs ta{};
        ta.queries = d_queries;
        ta.d = h.d;
        ta.nq = nq;
        ta.dims = x->dims.p;
        ta.sub = x->sub.p;
        ta.cent = x->cent.p;
        ta.cell_size = x->cell_size.p;  // GLOBAL cell sizes: the global Dynamic-Activation cut
        ta.ns = h.layout.ns;
        ta.k_half = h.p.k_half;
        ta.K = x->K;
        ta.hmax = x->hmax;
        ta.target = suco_collision_count(p->alpha, x->n_global);
        ta.cells = d_cells;
        ta.ncells = d_ncells;
        CUDA_TRY(launch_traverse(ta, st));
        x->launches = 1;  // a split-protocol round starts here (suco_gpu_last_launches)
    });
}

int suco_gpu_shard_histograms_cells(suco_gpu_index* x, uint64_t nq, const suco_collision_params* p,
                                    const uint32_t* d_cells, const uint64_t* d_cells_off, uint32_t* d_hist,
                                    void* stream) {
    return guarded([&] {
        if (!x) raise(SUCO_ERR_CONTRACT, "index is null");
        if (!x->dense) raise(SUCO_ERR_CONTRACT, "the _cells shard entry points need the dense select (N_s <= 8, blocks of 2048k ids)");
        validate_params(p, x->n_global);
        if (nq == 0) return;
        DeviceGuard g(x->device);
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : x->stream;
        auto& sl = x->slot[0];
        DenseArgs da = shard_dense_args(x, sl, nq);
        da.cells = d_cells;
        da.cells_off = d_cells_off;
        sl.dhist.reserve(nq * da.P * 8);
        da.hist = sl.dhist.p;
        CUDA_TRY(launch_dense_hist(da, st));
        CUDA_TRY(launch_dense_hist_rows(da, d_hist, st));
        x->launches += 2;
    });
}

int suco_gpu_shard_topk_cells(suco_gpu_index* x, const float* d_queries, uint64_t nq, uint32_t qlen,
                              const suco_collision_params* p, const uint32_t* d_cells, const uint64_t* d_cells_off,
                              const uint32_t* d_T, const uint32_t* d_quota, const uint32_t* d_base,
                              const uint32_t* d_counts, uint64_t stride, uint32_t* d_ids, double* d_sqdists,
                              void* stream) {
    return guarded([&] {
        if (!x) raise(SUCO_ERR_CONTRACT, "index is null");
        if (!x->dense) raise(SUCO_ERR_CONTRACT, "the _cells shard entry points need the dense select");
        if (qlen != x->host.d) raise(SUCO_ERR_CONTRACT, "query length does not match dataset d");
        validate_params(p, x->n_global);
        if (nq == 0) return;
        DeviceGuard g(x->device);
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : x->stream;
        const uint64_t sd = std::max<uint64_t>(stride, 1);
        x->shard_cands.reserve(nq * sd);
        DenseArgs da = shard_dense_args(x, x->slot[0], nq);
        da.cells = d_cells;
        da.cells_off = d_cells_off;
        da.m = sd;
        da.T = const_cast<uint32_t*>(d_T);
        da.quota = const_cast<uint32_t*>(d_quota);
        da.base = const_cast<uint32_t*>(d_base);
        da.cands = x->shard_cands.p;
        CUDA_TRY(launch_dense_emit(da, st));
        shard_rerank(x, d_queries, nq, p->k, d_counts, sd, d_ids, d_sqdists, st);
        x->launches += 1;
    });
}

int suco_gpu_shard_histograms(suco_gpu_index* x, const float* d_queries, uint64_t nq, uint32_t qlen,
                              const suco_collision_params* p, uint32_t* d_hist, void* stream) {
    return guarded([&] {
        if (!x) raise(SUCO_ERR_CONTRACT, "index is null");
        if (qlen != x->host.d) {
            raise(SUCO_ERR_CONTRACT, "query length " + std::to_string(qlen) + " does not match dataset d = " +
                                         std::to_string(x->host.d));
        }
        validate_params(p, x->n_global);
        if (nq == 0) return;
        DeviceGuard g(x->device);
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : x->stream;
        const uint64_t nl = x->host.n;
        const uint32_t ns = x->host.layout.ns;
        const uint32_t b = x->block ? x->block : static_cast<uint32_t>(nl);
        const uint32_t nblocks = static_cast<uint32_t>((nl + b - 1) / b);
        auto& sl = x->slot[0];
        if (x->dense) {  // traverse + dense piece histograms (dense.cu K1), in the exchange format
            stage_traverse(x, sl, d_queries, nq, suco_collision_count(p->alpha, x->n_global), st, nullptr);
            DenseArgs da = shard_dense_args(x, sl, nq);
            sl.dhist.reserve(nq * da.P * 8);
            da.hist = sl.dhist.p;
            CUDA_TRY(launch_dense_hist(da, st));
            CUDA_TRY(launch_dense_hist_rows(da, d_hist, st));
            x->phase1_nq = nq;
            return;
        }
        const uint64_t ss = (nl + 15) / 16 * 16;  // 16-byte score rows
        x->shard_scores.reserve(nq * ss);
        stage_traverse(x, sl, d_queries, nq, suco_collision_count(p->alpha, x->n_global), st, nullptr);
        sl.cands.reserve(1);
        SelectArgs sa{};
        sa.ids = x->ids.p;
        sa.slab_off = x->slab_off.p;
        sa.cells = sl.cells.p;
        sa.ncells = sl.ncells.p;
        sa.cells_cap = x->K;
        sa.n = nl;
        sa.ns = ns;
        sa.K = x->K;
        sa.nslabs = x->sel.nslabs;
        sa.CH = x->sel.CH;
        sa.rounds = x->sel.rounds;
        sa.CS = x->sel.CS;
        sa.m = 1;
        sa.nq = nq;
        sa.cands = sl.cands.p;
        sa.scores_dbg = x->shard_scores.p;
        sa.scores_stride = ss;
        sa.count_only = true;
        if (x->slab_is_block && x->sel.nslabs == nblocks) {
            sa.slab_hist = d_hist;
            CUDA_TRY(launch_select(sa, x->sel, nq, st));
        } else {
            CUDA_TRY(launch_select(sa, x->sel, nq, st));
            CUDA_TRY(launch_block_hist(x->shard_scores.p, nq, nl, ss, b, nblocks, ns, d_hist, st));
        }
    });
}

int suco_gpu_shard_topk(suco_gpu_index* x, const float* d_queries, uint64_t nq, uint32_t qlen,
                        const suco_collision_params* p, const uint32_t* d_T, const uint32_t* d_quota,
                        const uint32_t* d_base, const uint32_t* d_counts, uint64_t stride, uint32_t* d_ids,
                        double* d_sqdists, void* stream) {
    return guarded([&] {
        if (!x) raise(SUCO_ERR_CONTRACT, "index is null");
        if (qlen != x->host.d) raise(SUCO_ERR_CONTRACT, "query length does not match dataset d");
        validate_params(p, x->n_global);
        if (nq == 0) return;
        const uint64_t ss = (x->host.n + 15) / 16 * 16;
        if (x->dense ? x->phase1_nq != nq : x->shard_scores.cap < nq * ss) {
            raise(SUCO_ERR_CONTRACT, "suco_gpu_shard_topk needs phase 1 (suco_gpu_shard_histograms) of the same queries");
        }
        DeviceGuard g(x->device);
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : x->stream;
        const uint64_t nl = x->host.n;
        const uint32_t b = x->block ? x->block : static_cast<uint32_t>(nl);
        const uint32_t nblocks = static_cast<uint32_t>((nl + b - 1) / b);
        const uint64_t sd = std::max<uint64_t>(stride, 1);
        x->shard_cands.reserve(nq * sd);
        if (x->dense) {  // re-score each piece against the traversal of phase 1 (dense.cu K3)
            DenseArgs da = shard_dense_args(x, x->slot[0], nq);
            da.m = sd;
            da.T = const_cast<uint32_t*>(d_T);
            da.quota = const_cast<uint32_t*>(d_quota);
            da.base = const_cast<uint32_t*>(d_base);
            da.cands = x->shard_cands.p;
            CUDA_TRY(launch_dense_emit(da, st));
        } else {
            CUDA_TRY(launch_shard_emit(x->shard_scores.p, nq, nl, ss, b, nblocks, x->shard, x->num_shards, d_T, d_quota,
                                       d_base, x->shard_cands.p, sd, st));
        }
        shard_rerank(x, d_queries, nq, p->k, d_counts, sd, d_ids, d_sqdists, st);
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
            if (h[0] == 0 && h[2] == 0 && mx <= 255.f && d <= 512 && !std::getenv("SUCO_NO_U8")) {
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

// ------------------------------------------------------------------ vecs I/O (io.cpp:99-210)
// Record framing shared by fvecs / bvecs / ivecs: [dim i32 LE][dim elements]. Parsed in order
// with the reference's checks and messages (io.cpp:46-85, 99-137), so the first error wins
// exactly as there. Rows stream through two pinned staging buffers straight into device memory.
namespace {

constexpr int32_t kVecsMaxDim = 1 << 20;
constexpr double kVecsMaxExactInt = 16777216.0;  // 2^24

size_t vecs_elem(int kind) { return kind == 1 ? 1 : 4; }

uint32_t le32(const unsigned char* p) {
    return uint32_t(p[0]) | (uint32_t(p[1]) << 8) | (uint32_t(p[2]) << 16) | (uint32_t(p[3]) << 24);
}

struct VecsFile {
    FILE* f = nullptr;
    uint64_t size = 0;
    ~VecsFile() {
        if (f) std::fclose(f);
    }
};

void vecs_open(VecsFile& vf, const std::string& path) {
    vf.f = std::fopen(path.c_str(), "rb");
    if (!vf.f) raise(SUCO_ERR_FORMAT, "cannot open file: " + path);
    std::fseek(vf.f, 0, SEEK_END);
    vf.size = static_cast<uint64_t>(std::ftell(vf.f));
    std::fseek(vf.f, 0, SEEK_SET);
    if (vf.size == 0) raise(SUCO_ERR_FORMAT, "empty file: " + path);
}

// Streams records [0, limit) through `sink(first_record, count, float rows)`; returns n, sets d.
template <typename Sink>
uint64_t vecs_stream(const std::string& path, int kind, uint64_t limit, uint32_t& d, float* stage_a, float* stage_b,
                     uint64_t stage_rows, Sink&& sink) {
    VecsFile vf;
    vecs_open(vf, path);
    const size_t es = vecs_elem(kind);
    std::vector<unsigned char> buf;
    uint64_t pos = 0, record = 0;
    d = 0;
    float* stage[2] = {stage_a, stage_b};
    int which = 0;
    uint64_t in_stage = 0, stage_first = 0;
    while (pos < vf.size && record < limit) {
        unsigned char hdr[4];
        if (vf.size - pos < 4) {
            raise(SUCO_ERR_FORMAT, path + ": truncated record header at byte offset " + std::to_string(pos) +
                                       " (record " + std::to_string(record) + ")");
        }
        if (std::fread(hdr, 1, 4, vf.f) != 4) raise(SUCO_ERR_FORMAT, "failed reading file: " + path);
        const int32_t dim = static_cast<int32_t>(le32(hdr));
        if (dim <= 0 || dim > kVecsMaxDim) {
            raise(SUCO_ERR_FORMAT, path + ": record " + std::to_string(record) + " declares invalid dimension " +
                                       std::to_string(dim));
        }
        if (record == 0) {
            d = static_cast<uint32_t>(dim);
            buf.resize(size_t(d) * es);
        } else if (static_cast<uint32_t>(dim) != d) {
            raise(SUCO_ERR_FORMAT, path + ": record " + std::to_string(record) + " has dimension " +
                                       std::to_string(dim) + ", expected " + std::to_string(d));
        }
        pos += 4;
        const uint64_t body = uint64_t(dim) * es;
        if (vf.size - pos < body) {
            raise(SUCO_ERR_FORMAT, path + ": truncated record body at byte offset " + std::to_string(pos) +
                                       " (record " + std::to_string(record) + ")");
        }
        if (std::fread(buf.data(), 1, body, vf.f) != body) raise(SUCO_ERR_FORMAT, "failed reading file: " + path);
        float* row = stage[which] + in_stage * d;
        for (uint32_t j = 0; j < d; ++j) {
            float v = 0.f;
            if (kind == 0) {
                const uint32_t bits = le32(buf.data() + 4 * size_t(j));
                std::memcpy(&v, &bits, 4);
                if (!std::isfinite(v)) {
                    raise(SUCO_ERR_FORMAT, path + ": non-finite value in record " + std::to_string(record));
                }
            } else if (kind == 1) {
                v = static_cast<float>(buf[j]);
            } else {
                const int32_t iv = static_cast<int32_t>(le32(buf.data() + 4 * size_t(j)));
                if (iv > int32_t(kVecsMaxExactInt) || iv < -int32_t(kVecsMaxExactInt)) {
                    raise(SUCO_ERR_FORMAT, path + ": record " + std::to_string(record) + " holds " +
                                               std::to_string(iv) + ", too large to load into floats exactly");
                }
                v = static_cast<float>(iv);
            }
            row[j] = v;
        }
        pos += body;
        ++record;
        if (++in_stage == stage_rows) {
            sink(stage_first, in_stage, stage[which], which);
            which ^= 1;
            stage_first = record;
            in_stage = 0;
        }
    }
    if (record == 0) raise(SUCO_ERR_FORMAT, path + ": no records within the read limit");
    if (in_stage) sink(stage_first, in_stage, stage[which], which);
    return record;
}

// Upper bound on the records of a vecs file (for the device allocation): every record has the
// first record's dim. Exact unless the file is malformed (then the parse raises anyway).
uint64_t vecs_bound(const std::string& path, int kind, uint64_t limit, uint32_t* dim) {
    VecsFile vf;
    vecs_open(vf, path);
    unsigned char hdr[4];
    if (vf.size < 4 || std::fread(hdr, 1, 4, vf.f) != 4) {
        raise(SUCO_ERR_FORMAT, path + ": truncated record header at byte offset 0 (record 0)");
    }
    const int32_t d0 = static_cast<int32_t>(le32(hdr));
    if (d0 <= 0 || d0 > kVecsMaxDim) {
        raise(SUCO_ERR_FORMAT, path + ": record 0 declares invalid dimension " + std::to_string(d0));
    }
    *dim = static_cast<uint32_t>(d0);
    const uint64_t stride = 4 + uint64_t(d0) * vecs_elem(kind);
    const uint64_t n = (vf.size + stride - 1) / stride;
    return std::min(n, limit);
}

void check_kind(int kind) {
    if (kind < 0 || kind > 2) raise(SUCO_ERR_CONTRACT, "vecs kind must be 0 (fvecs), 1 (bvecs) or 2 (ivecs)");
}

// Streams a vecs file into x->data (n x d f32 on the device).
void stream_vecs_into(suco_gpu_index* x, const std::string& path, int kind, uint64_t limit, uint64_t* n_out,
                      uint32_t* d_out) {
    uint32_t d0 = 0;
    const uint64_t nmax = vecs_bound(path, kind, limit, &d0);
    x->data.reserve(nmax * d0);
    const uint64_t rows = std::max<uint64_t>(1, (32ull << 20) / (uint64_t(d0) * 4));  // 32 MB stages
    float* pin[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    try {
        for (int i = 0; i < 2; ++i) {
            CUDA_TRY(cudaMallocHost(&pin[i], rows * d0 * 4));
            CUDA_TRY(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
            CUDA_TRY(cudaEventRecord(done[i], x->stream));
        }
        uint32_t d = 0;
        // a stage is refilled only after its previous copy finished (event), so parsing the next
        // chunk overlaps the copy of the last one
        auto wait_stage = [&](int w) { CUDA_TRY(cudaEventSynchronize(done[w])); };
        wait_stage(0);
        const uint64_t n = vecs_stream(path, kind, limit, d, pin[0], pin[1], rows,
                                       [&](uint64_t first, uint64_t cnt, const float* rowsp, int w) {
            CUDA_TRY(cudaMemcpyAsync(x->data.p + first * d, rowsp, cnt * d * 4, cudaMemcpyHostToDevice, x->stream));
            CUDA_TRY(cudaEventRecord(done[w], x->stream));
            wait_stage(w ^ 1);
        });
        CUDA_TRY(cudaStreamSynchronize(x->stream));
        *n_out = n;
        *d_out = d;
    } catch (...) {
        for (int i = 0; i < 2; ++i) {
            if (pin[i]) cudaFreeHost(pin[i]);
            if (done[i]) cudaEventDestroy(done[i]);
        }
        throw;
    }
    for (int i = 0; i < 2; ++i) {
        cudaFreeHost(pin[i]);
        cudaEventDestroy(done[i]);
    }
}

}  // namespace

int suco_read_vecs(const char* path, int kind, uint64_t limit, float* out, uint64_t cap_rows, uint64_t* n,
                   uint32_t* d) {
    return guarded([&] {
        if (!path || !n || !d) raise(SUCO_ERR_CONTRACT, "null argument");
        check_kind(kind);
        if (!out) {  // size query: parse the framing, keep nothing
            uint32_t dd = 0;
            const uint64_t rows = 4096;
            std::vector<float> a, b;
            uint32_t d0 = 0;
            vecs_bound(path, kind, limit, &d0);
            a.resize(rows * d0);
            b.resize(rows * d0);
            *n = vecs_stream(path, kind, limit, dd, a.data(), b.data(), rows, [](uint64_t, uint64_t, const float*, int) {});
            *d = dd;
            return;
        }
        uint32_t d0 = 0;
        vecs_bound(path, kind, limit, &d0);
        const uint64_t rows = 4096;
        std::vector<float> a(rows * d0), b(rows * d0);
        uint32_t dd = 0;
        *n = vecs_stream(path, kind, limit, dd, a.data(), b.data(), rows,
                         [&](uint64_t first, uint64_t cnt, const float* rowsp, int) {
            if (first + cnt > cap_rows) raise(SUCO_ERR_CONTRACT, "output buffer holds fewer rows than the file");
            std::memcpy(out + first * dd, rowsp, cnt * dd * 4);
        });
        *d = dd;
    });
}

int suco_write_vecs(const char* path, int kind, uint64_t n, uint32_t d, const float* values) {
    return guarded([&] {
        if (!path || !values) raise(SUCO_ERR_CONTRACT, "null argument");
        check_kind(kind);
        if (n < 1 || d < 1) raise(SUCO_ERR_CONTRACT, "write_vecs: n and d must be >= 1");
        std::vector<unsigned char> rec(4 + size_t(d) * vecs_elem(kind));
        rec[0] = static_cast<unsigned char>(d);
        rec[1] = static_cast<unsigned char>(d >> 8);
        rec[2] = static_cast<unsigned char>(d >> 16);
        rec[3] = static_cast<unsigned char>(d >> 24);
        for (uint64_t i = 0; i < n * d; ++i) {  // validate before touching the file (io.cpp:139-160)
            const float v = values[i];
            if (kind == 1 && !(v == std::trunc(v) && v >= 0.f && v <= 255.f)) {
                raise(SUCO_ERR_CONTRACT, "write_vecs: bvecs values must be integers in [0, 255]");
            }
            if (kind == 2 && !(v == std::trunc(v) && std::fabs(v) <= kVecsMaxExactInt)) {
                raise(SUCO_ERR_CONTRACT, "write_vecs: ivecs values must be integers with |v| <= 2^24");
            }
        }
        FILE* f = std::fopen(path, "wb");
        if (!f) raise(SUCO_ERR_INTERNAL, std::string("cannot open file for writing: ") + path);
        bool ok = true;
        for (uint64_t r = 0; r < n && ok; ++r) {
            for (uint32_t j = 0; j < d; ++j) {
                const float v = values[r * d + j];
                if (kind == 0) {
                    std::memcpy(rec.data() + 4 + 4 * size_t(j), &v, 4);
                } else if (kind == 1) {
                    rec[4 + j] = static_cast<unsigned char>(v);
                } else {
                    const int32_t iv = static_cast<int32_t>(v);
                    std::memcpy(rec.data() + 4 + 4 * size_t(j), &iv, 4);
                }
            }
            ok = std::fwrite(rec.data(), 1, rec.size(), f) == rec.size();
        }
        ok = (std::fclose(f) == 0) && ok;
        if (!ok) raise(SUCO_ERR_INTERNAL, std::string("failed writing file: ") + path);
    });
}

int suco_gpu_build_index_from_vecs(const char* path, int kind, uint64_t limit, const suco_index_params* params,
                                   int device, suco_gpu_index** out) {
    return guarded([&] {
        if (!out || !path) raise(SUCO_ERR_CONTRACT, "null argument");
        *out = nullptr;
        if (!params) raise(SUCO_ERR_CONTRACT, "index params are null");
        check_kind(kind);
        DeviceGuard g(device);
        suco_gpu_index* x = new_index(device);
        try {
            create_stream(x);
            uint64_t n = 0;
            uint32_t d = 0;
            stream_vecs_into(x, path, kind, limit, &n, &d);
            upload_data(x, nullptr, n, d);
            build_core(x, n, d, params);
        } catch (...) {
            delete x;
            throw;
        }
        *out = x;
    });
}

int suco_gpu_load_index_from_vecs(const unsigned char* bytes, uint64_t len, const char* path, int kind, uint64_t limit,
                                  int device, suco_gpu_index** out) {
    return guarded([&] {
        if (!out || !path) raise(SUCO_ERR_CONTRACT, "null argument");
        *out = nullptr;
        HostIndex h = parse_index(bytes, len);  // FORMAT first, like load_index + read_vecs in suco_cli.cpp:241-244
        check_kind(kind);
        DeviceGuard g(device);
        suco_gpu_index* x = new_index(device);
        try {
            create_stream(x);
            uint64_t n = 0;
            uint32_t d = 0;
            stream_vecs_into(x, path, kind, limit, &n, &d);
            if (h.n != n) {
                raise(SUCO_ERR_INCOMPATIBLE, "index was built from n = " + std::to_string(h.n) +
                                                 " points but dataset has n = " + std::to_string(n));
            }
            if (h.d != d) {
                raise(SUCO_ERR_INCOMPATIBLE, "index was built for d = " + std::to_string(h.d) +
                                                 " but dataset has d = " + std::to_string(d));
            }
            x->host = std::move(h);
            upload_data(x, nullptr, n, d);
            load_core(x, n);
        } catch (...) {
            delete x;
            throw;
        }
        *out = x;
    });
}
