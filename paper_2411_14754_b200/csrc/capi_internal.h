// Internals shared by the C-ABI translation units (capi*.cu): the opaque
// handle types of include/suco_b200.h, device buffers, error mapping.
//
// Threading model (the reference's, index.hpp:63-66 + query.hpp:72-78): an
// index handle is immutable once built or loaded — every query reads it and
// nothing on it changes — and all per-call state (scratch, streams, events,
// profiling counters) lives in a suco_gpu_query_ctx, which mirrors the
// reference's caller-owned QueryScratch. Calls that take no context borrow
// one from the index's pool (mutex-guarded check-out / check-in), so any
// number of host threads may query one index at once.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/suco_b200.h"
#include "index_format.h"
#include "kernels.h"
#include "tuning.h"

namespace suco_gpu {

extern thread_local std::string g_err;

// A failed device allocation: the query pipeline retries with smaller tiles.
struct OutOfDeviceMemory {};

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
    } catch (const OutOfDeviceMemory&) {
        g_err = "out of device memory";
        return SUCO_ERR_INTERNAL;
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
        const cudaError_t e = cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T));
        if (e == cudaErrorMemoryAllocation) {
            cudaGetLastError();
            p = nullptr;
            throw OutOfDeviceMemory{};
        }
        CUDA_TRY(e);
        cap = count;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    size_t bytes() const { return cap * sizeof(T); }
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
};

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev);
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// Owned non-blocking stream (stand-alone calls that must not share one).
struct OwnStream {
    cudaStream_t s = nullptr;
    OwnStream();
    ~OwnStream() {
        if (s) cudaStreamDestroy(s);
    }
};

void validate_params(const suco_collision_params* p, uint64_t n);
void check_query_len(uint32_t qlen, uint32_t d);

}  // namespace suco_gpu

// Per-call query state (the reference's QueryScratch, query.hpp:72-78): the
// tile scratch of the three-stage pipeline, its streams and events, and the
// profiling counters of the last call. Bound to one index.
struct suco_gpu_query_ctx {
    const suco_gpu_index* index = nullptr;
    int device = 0;
    cudaStream_t own = nullptr;  // the context's default stream (NULL stream arguments)
    // query pipeline: tiles flow traverse -> select -> rerank on three streams,
    // double-buffered scratch, so neighbouring tiles overlap on the device.
    struct Slot {
        suco_gpu::DevBuf<float> q;
        suco_gpu::DevBuf<uint32_t> cells, ncells, cands, out_ids, all_id;
        suco_gpu::DevBuf<uint16_t> dhist;               // dense select: nq x P x 8
        suco_gpu::DevBuf<uint32_t> dT, dquota, dbase;   // dense select plan
        suco_gpu::DevBuf<uint16_t> dsample;             // single-pass select: sampled histograms
        suco_gpu::DevBuf<uint16_t> dcbuf, dccnt;        // single-pass select: candidate buffers and their counts
        suco_gpu::DevBuf<uint32_t> dL, dflag, dh2;      // single-pass select: bound, fallback flags, two-level counts
        suco_gpu::DevBuf<double> out_d, all_d;
        cudaEvent_t trav = nullptr, sel = nullptr, rr = nullptr;
        cudaEvent_t selmain = nullptr;  // dense select: every unflagged query's candidates written
        size_t bytes() const {
            return q.bytes() + cells.bytes() + ncells.bytes() + cands.bytes() + out_ids.bytes() + all_id.bytes() +
                   dhist.bytes() + dT.bytes() + dquota.bytes() + dbase.bytes() + dsample.bytes() + dcbuf.bytes() +
                   dccnt.bytes() + dL.bytes() + dflag.bytes() + dh2.bytes() + out_d.bytes() + all_d.bytes();
        }
        void release_all();
    };
    Slot slot[2];
    cudaStream_t pipe[4] = {nullptr, nullptr, nullptr, nullptr};  // traverse, select, rerank, fallback
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    // shard protocol scratch (capi_shard.cu)
    suco_gpu::DevBuf<uint32_t> sh_tot, sh_tot_all, sh_ties, sh_ties_all, sh_qblk, sh_counts, sh_ids, sh_ids_all;
    suco_gpu::DevBuf<uint32_t> sh_s17, sh_gt, sh_gts, sh_nflag;  // shard single pass: sampled totals, #(> L), flags
    suco_gpu::DevBuf<uint64_t> sh_need;
    suco_gpu::DevBuf<double> sh_sq, sh_sq_all;
    uint64_t exchange_bytes = 0;  // bytes this rank sent through the communicator in the last call
    uint64_t budget = 0;          // scratch budget (bytes): set on first use from free memory, halved on OOM
    uint64_t sh_key[3] = {0, 0, 0}, sh_tiles = 0;  // shard tile count agreed for (nq, m, k)
    // stage profiling (suco_gpu_query_ctx_set_profiling)
    bool profile = false;
    std::vector<cudaEvent_t> events;  // pairs (start, end) per profiled stage launch
    std::vector<int> event_stage;     // stage of each pair
    uint32_t pairs = 0;
    suco_gpu::DevBuf<unsigned long long> stat_cum;
    uint64_t last_nq = 0, last_m = 0;
    uint64_t launches = 0;  // kernels enqueued by the last query call

    ~suco_gpu_query_ctx();
};

struct suco_gpu_index {
    int device = 0;
    cudaStream_t own = nullptr;  // build / upload stream (queries run on their context's streams)
    suco_gpu::Tuning tune;       // read once at creation (tuning.h)
    suco_gpu::HostIndex host;    // layout, params, centroids (IMI lives on the device)
    uint32_t K = 0, hmax = 0;
    suco_gpu::DevBuf<float> data;
    suco_gpu::DevBuf<uint32_t> dims;
    suco_gpu::DevBuf<suco_gpu::SubDesc> sub;
    suco_gpu::DevBuf<float> cent;
    suco_gpu::DevBuf<uint32_t> cell_off;   // ns x (K+1)
    suco_gpu::DevBuf<uint32_t> cell_size;  // ns x K (GLOBAL sizes on a shard)
    suco_gpu::DevBuf<uint32_t> ids;        // ns x n
    suco_gpu::DevBuf<uint32_t> slab_off;   // ns x K x (nslabs+1)
    suco_gpu::SelectConfig sel{};
    float data_int_max = -1.f;  // integer certificate of the dataset (rerank fp32 path)
    suco_gpu::DevBuf<uint8_t> data8;   // u8 copy of the rows when they are integers in [0, 255] (rerank u8 path)
    suco_gpu::DevBuf<int8_t> q8;       // int8 screen records of float rows (n x qrec; rerank_q8_kernel)
    uint32_t qpad = 0, qrec = 0;       // int8 bytes / record stride (0: no int8 copy)
    uint32_t qpre = 0, qsplit = 0;     // prefix-bound record layout (pack_q8_kernel)
    uint64_t q8_rows = 0;              // rows in q8 (the rests of prefix-bound records start at q8_rows * qsplit)
    suco_gpu::DevBuf<uint16_t> codes;  // n x 8: s*K + cell of every point (dense select, N_s <= 8)
    bool dense = false;         // select stage = dense bit-sliced 32-query blocks (dense.cu)
    bool dense_hgroup = false;  // ... with the interleaved table (eight subspaces, not the cluster-pair pass)
    bool dense_half = false;    // ... in the half-width mode (16-query blocks, u16 masks; large N_s*K)
    uint32_t dpad = 0;          // row bytes of data8 (0: no u8 copy)
    // block-cyclic shard: global blocks j with j % num_shards == shard
    uint32_t shard = 0, num_shards = 1, block = 0;
    uint64_t n_global = 0;      // dataset size the index describes (== host.n unsharded)
    // pool of query contexts for calls that bring none (mutable: check-out / check-in only)
    mutable std::mutex pool_mu;
    mutable std::vector<suco_gpu_query_ctx*> pool;

    ~suco_gpu_index();
};

namespace suco_gpu {

// Context lifecycle (capi.cu).
suco_gpu_query_ctx* ctx_new(const suco_gpu_index* x);
// RAII check-out of a pooled context (or the caller's).
struct CtxLease {
    const suco_gpu_index* x;
    suco_gpu_query_ctx* c;
    bool pooled;
    CtxLease(const suco_gpu_index* x, suco_gpu_query_ctx* given);
    ~CtxLease();
};
void check_ctx(const suco_gpu_index* x, const suco_gpu_query_ctx* c);

// Pipeline pieces shared with the shard protocol (capi.cu).
void begin_call(suco_gpu_query_ctx* c, uint64_t nq, uint64_t m, cudaStream_t st);
void stage_traverse(const suco_gpu_index* x, suco_gpu_query_ctx* c, suco_gpu_query_ctx::Slot& sl, const float* d_q,
                    uint64_t nt, uint64_t target, cudaStream_t st, double* dbg_sum, uint64_t* dbg_cum, bool profiled);
DenseArgs dense_args(const suco_gpu_index* x, suco_gpu_query_ctx::Slot& sl, uint64_t nq);
// points per piece of the dense single pass for n points and nq queries (qper queries per CTA)
uint32_t fused_piece(uint64_t n, uint64_t nq, uint32_t qper);
void rerank_args(const suco_gpu_index* x, RerankArgs& ra);

// Device upload pieces shared by build / load / shard (capi.cu).
suco_gpu_index* new_index_on(int device);  // tuning read from the environment, own stream created
void upload_data(suco_gpu_index* x, const float* data, uint64_t n, uint32_t d);
void build_core(suco_gpu_index* x, uint64_t n, uint32_t d, const suco_index_params* params,
                const uint32_t* train = nullptr, uint64_t n_train = 0);
void load_core(suco_gpu_index* x, uint64_t n);
void create_index_stream(suco_gpu_index* x);
void upload_codebooks(suco_gpu_index* x);
void set_l2_persisting(const suco_gpu_index* x);
void apply_l2_window(const suco_gpu_index* x, cudaStream_t st);
void finalize_dense(suco_gpu_index* x, bool allow_half);

}  // namespace suco_gpu
