// Stage 3 of the query path: exact re-rank of the candidate rows and top-k
// (query.cpp:159-197): squared distance with the reference's 4-accumulator
// fp64 kernel over the full d, top-k by (squared distance, id), sqrt last.
//
// One CTA (8 warps) per query; the query row is staged once as doubles in
// shared memory. A warp re-ranks 8 candidate rows per step: the 8 rows are
// gathered with coalesced 16-byte loads (one 512-byte row per warp-load at
// d = 128) into a padded shared tile, then lane (r, a) = (lane/4, lane%4)
// folds accumulator a of row r in index order — exactly the reference's
// acc0..acc3 chains — and the four partials combine as (a0+a1)+(a2+a3).
// The tile stride of 132 floats makes both the row stores and the strided
// chain reads bank-conflict free. Each warp keeps a sorted top-k (k <= 32)
// in registers, one entry per lane; warps merge through shared memory.
// k > 32 writes every (dist, id) to scratch and a second kernel selects.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace suco_gpu {
namespace {

constexpr uint32_t kWarps = 8;
constexpr uint32_t kThreads = 32 * kWarps;
constexpr uint32_t kRows = 8;     // rows per warp step
constexpr uint32_t kChunk = 128;  // dims per staged chunk
constexpr uint32_t kStride = 132; // padded tile row (floats)
constexpr uint32_t kFull = 0xffffffffu;

// This CTA's query: blockIdx.x, minus the queries `qskip` marks (their candidates are not ready
// yet), or the blockIdx.x-th entry of `qlist` (a later pass over exactly those queries).
// false: the CTA has no query.
__device__ __forceinline__ bool rerank_query(const RerankArgs& a, uint64_t& q) {
    if (a.qlist) {
        if (blockIdx.x >= *a.nlist) return false;
        q = a.qlist[blockIdx.x];
        return true;
    }
    q = blockIdx.x;
    return !(a.qskip && a.qskip[q]);
}

__device__ __forceinline__ float4 ld_stream4(const float* p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}

__device__ __forceinline__ bool is_u8(float v) { return v == truncf(v) && v >= 0.f && v <= 255.f; }

// Inserts (d, id) into the warp's sorted list (lane i holds entry i, k <= 32).
__device__ __forceinline__ void warp_insert(double d, uint32_t id, double& ld, uint32_t& lid, uint32_t k,
                                            uint32_t lane) {
    const double wd = __shfl_sync(kFull, ld, k - 1);
    const uint32_t wi = __shfl_sync(kFull, lid, k - 1);
    if (!dist_id_less(d, id, wd, wi)) return;  // warp-uniform
    const bool less = lane < k && dist_id_less(ld, lid, d, id);
    const uint32_t pos = __popc(__ballot_sync(kFull, less));
    const double ud = __shfl_up_sync(kFull, ld, 1);
    const uint32_t ui = __shfl_up_sync(kFull, lid, 1);
    if (lane > pos) {
        ld = ud;
        lid = ui;
    } else if (lane == pos) {
        ld = d;
        lid = id;
    }
}

template <bool VEC, bool GENERIC>
__global__ void __launch_bounds__(kThreads) rerank_kernel(RerankArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    double* qd = reinterpret_cast<double*>(smem);                                  // d
    float* qf = reinterpret_cast<float*>(smem + ((a.d * 8 + 15) / 16) * 16);       // d
    float* tile = qf + ((a.d + 3) / 4) * 4;                                          // warps x rows x stride
    __shared__ unsigned int qstat[2];
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    uint64_t q;
    if (!rerank_query(a, q)) return;
    const float* query = a.queries + q * a.d;
    if (tid < 2) qstat[tid] = 0;
    __syncthreads();
    bool qbad = false, qu8 = true;
    float qmax = 0.f;
    for (uint32_t i = tid; i < a.d; i += kThreads) {
        const float v = query[i];
        qd[i] = static_cast<double>(v);
        qf[i] = v;
        qbad |= (v != truncf(v));
        qu8 &= is_u8(v);
        qmax = fmaxf(qmax, fabsf(v));
    }
    if (a.data8 && __syncthreads_and(qu8)) return;  // rerank_u8_kernel owns this query
    qbad = __any_sync(kFull, qbad);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) qmax = fmaxf(qmax, __shfl_xor_sync(kFull, qmax, o));
    if (lane == 0) {
        if (qbad) atomicOr(&qstat[0], 1u);
        atomicMax(&qstat[1], __float_as_uint(qmax));
    }
    __syncthreads();
    // Certified-exact fp32 chains: with integer data and query, every term
    // (a-b)^2 and every partial sum of a chain is an integer below 2^24, so
    // fp32 FFMA reproduces the reference's fp64 chain values bit for bit.
    bool use32 = false;
    if (a.data_int_max >= 0.f && qstat[0] == 0) {
        const double span = static_cast<double>(a.data_int_max) + static_cast<double>(__uint_as_float(qstat[1]));
        use32 = (static_cast<double>(a.d / 4 + 4) * span * span) < 16777216.0;
    }

    float* wt = tile + warp * kRows * kStride;
    const uint32_t r = lane >> 2, acc_i = lane & 3u;
    const uint32_t main4 = a.d & ~3u;  // dims covered by the four chains
    const uint32_t* cands = a.cands + q * a.m;
    const uint64_t mq = a.counts ? a.counts[q] : a.m;
    double ld = kInf;
    uint32_t lid = 0xffffffffu;

    for (uint64_t base = static_cast<uint64_t>(warp) * kRows; base < mq; base += kRows * kWarps) {
        // candidate ids of the 8 rows (lanes 0..7 load, broadcast); `gid` is the
        // reported id, `rid` the row in `data` (differs on shards)
        uint32_t my_id = 0;
        if (lane < kRows && base + lane < mq) {
            my_id = a.identity ? static_cast<uint32_t>(base + lane) : __ldcs(cands + base + lane);  // read once
        }
        uint32_t gid[kRows], rid[kRows];
#pragma unroll
        for (uint32_t j = 0; j < kRows; ++j) {
            gid[j] = __shfl_sync(kFull, my_id, j);
            rid[j] = gid[j];
        }
        const uint32_t nrows = static_cast<uint32_t>(min_u64(kRows, mq - base));
        double acc = 0.0;
        float acc32 = 0.f;
        for (uint32_t c0 = 0; c0 < a.d; c0 += kChunk) {
            const uint32_t cl = min(kChunk, a.d - c0);
            if constexpr (VEC) {
                float4 v[kRows];
#pragma unroll
                for (uint32_t j = 0; j < kRows; ++j) {
                    if (j < nrows && 4 * lane < cl) v[j] = ld_stream4(a.data + static_cast<uint64_t>(rid[j]) * a.d + c0 + 4 * lane);
                }
#pragma unroll
                for (uint32_t j = 0; j < kRows; ++j) {
                    if (j < nrows && 4 * lane < cl) *reinterpret_cast<float4*>(wt + j * kStride + 4 * lane) = v[j];
                }
            } else {
#pragma unroll
                for (uint32_t j = 0; j < kRows; ++j) {
                    if (j < nrows) {
                        const float* src = a.data + static_cast<uint64_t>(rid[j]) * a.d + c0;
                        for (uint32_t e = lane; e < cl; e += 32) wt[j * kStride + e] = __ldg(src + e);
                    }
                }
            }
            __syncwarp();
            if (r < nrows) {
                const float* row = wt + r * kStride;
                // chain acc_i over global dims c0 + 4t + acc_i < main4, in order
                const uint32_t lim = main4 > c0 ? min(cl, main4 - c0) : 0u;
                if (use32) {
#pragma unroll 8
                    for (uint32_t e = acc_i; e < lim; e += 4) {
                        const float df = row[e] - qf[c0 + e];
                        acc32 = __fmaf_rn(df, df, acc32);
                    }
                } else {
#pragma unroll 8
                    for (uint32_t e = acc_i; e < lim; e += 4) acc = __dadd_rn(acc, sqdiff_d(row[e], qd[c0 + e]));
                }
            }
            __syncwarp();
        }
        if (use32) acc = static_cast<double>(acc32);  // exact integer
        // tail dims (d % 4) fold into acc0 after its main chain (core.hpp:79-82)
        if (acc_i == 0 && r < nrows && main4 < a.d) {
            const float* src = a.data + static_cast<uint64_t>(rid[r]) * a.d;
            for (uint32_t g = main4; g < a.d; ++g) acc = __dadd_rn(acc, sqdiff_d(__ldg(src + g), qd[g]));
        }
        const double a1 = __shfl_down_sync(kFull, acc, 1);
        const double a2 = __shfl_down_sync(kFull, acc, 2);
        const double a3 = __shfl_down_sync(kFull, acc, 3);
        const double dist = __dadd_rn(__dadd_rn(acc, a1), __dadd_rn(a2, a3));  // valid on lanes 4r
        if constexpr (GENERIC) {
            if (acc_i == 0 && r < nrows) {
                a.all_d[q * a.m + base + r] = dist;
                a.all_id[q * a.m + base + r] = gid[r];
            }
        } else {
#pragma unroll
            for (uint32_t j = 0; j < kRows; ++j) {
                const double dj = __shfl_sync(kFull, dist, 4 * j);
                if (j < nrows) warp_insert(dj, gid[j], ld, lid, a.k, lane);
            }
        }
    }
    if constexpr (!GENERIC) {
        // merge the 8 warp lists through shared memory (reuse the tile area)
        __syncthreads();
        double* md = reinterpret_cast<double*>(tile);
        uint32_t* mi = reinterpret_cast<uint32_t*>(md + kWarps * 32);
        md[warp * 32 + lane] = ld;
        mi[warp * 32 + lane] = lid;
        __syncthreads();
        if (warp == 0) {
            for (uint32_t w = 1; w < kWarps; ++w) {
                for (uint32_t i = 0; i < a.k; ++i) {
                    const double dv = md[w * 32 + i];
                    if (dv == kInf) break;
                    warp_insert(dv, mi[w * 32 + i], ld, lid, a.k, lane);
                }
            }
            if (lane < a.k) {
                a.out_ids[q * a.k + lane] = lid;
                a.out_dists[q * a.k + lane] = a.squared ? ld : __dsqrt_rn(ld);
            }
        }
    }
}

// ------------------------------------------------------- pipelined f32 rows
// The same arithmetic as rerank_kernel (rows d % 4 == 0), with the row gathers moved off the
// critical path: a warp's work is a sequence of items (8-row group, 128-dim chunk); each item is
// copied global -> shared with 16-byte cp.async into one of kStages ring slots, kStages - 1 items
// ahead of the one being folded, and the candidate ids of the next kIdAhead groups are loaded
// into the warp's registers (lane 8t + j holds id j of group g with g % kIdAhead == t) long
// before their rows are requested. One CTA per query, 2 CTAs per SM.
constexpr uint32_t kStages = 3;
constexpr uint32_t kIdAhead = 4;

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <bool GENERIC>
__global__ void __launch_bounds__(kThreads, 2) rerank_pipe_kernel(RerankArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    double* qd = reinterpret_cast<double*>(smem);                             // d
    float* qf = reinterpret_cast<float*>(smem + ((a.d * 8 + 15) / 16) * 16);  // d
    float* ring = qf + ((a.d + 3) / 4) * 4;                                     // warps x stages x rows x stride
    __shared__ unsigned int qstat[2];
    __shared__ uint32_t idbuf[kWarps][kStages][kRows];  // the ids of each ring slot's rows
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    uint64_t q;
    if (!rerank_query(a, q)) return;
    const float* query = a.queries + q * a.d;
    if (tid < 2) qstat[tid] = 0;
    __syncthreads();
    bool qbad = false, qu8 = true;
    float qmax = 0.f;
    for (uint32_t i = tid; i < a.d; i += kThreads) {
        const float v = query[i];
        qd[i] = static_cast<double>(v);
        qf[i] = v;
        qbad |= (v != truncf(v));
        qu8 &= is_u8(v);
        qmax = fmaxf(qmax, fabsf(v));
    }
    if (a.data8 && __syncthreads_and(qu8)) return;  // rerank_u8_kernel owns this query
    qbad = __any_sync(kFull, qbad);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) qmax = fmaxf(qmax, __shfl_xor_sync(kFull, qmax, o));
    if (lane == 0) {
        if (qbad) atomicOr(&qstat[0], 1u);
        atomicMax(&qstat[1], __float_as_uint(qmax));
    }
    __syncthreads();
    bool use32 = false;  // certified-exact fp32 chains (see rerank_kernel)
    if (a.data_int_max >= 0.f && qstat[0] == 0) {
        const double span = static_cast<double>(a.data_int_max) + static_cast<double>(__uint_as_float(qstat[1]));
        use32 = (static_cast<double>(a.d / 4 + 4) * span * span) < 16777216.0;
    }

    float* wr = ring + warp * kStages * kRows * kStride;
    const uint32_t r = lane >> 2, acc_i = lane & 3u;
    const uint32_t* cands = a.cands + q * a.m;
    const uint64_t mq = a.counts ? a.counts[q] : a.m;
    const uint32_t nch = (a.d + kChunk - 1) / kChunk;
    const uint64_t first = uint64_t(warp) * kRows;
    const uint64_t groups = mq > first ? (mq - first + kRows * kWarps - 1) / (kRows * kWarps) : 0;
    const uint64_t items = groups * nch;
    auto gbase = [&](uint64_t g) { return first + g * kRows * kWarps; };
    auto load_id = [&](uint64_t g) -> uint32_t {  // this lane's id slot of group g
        const uint64_t i = gbase(g) + (lane & 7u);
        if (g >= groups || i >= mq) return 0u;
        return a.identity ? static_cast<uint32_t>(i) : __ldcs(cands + i);
    };
    uint32_t idreg = 0;
#pragma unroll
    for (uint32_t t = 0; t < kIdAhead; ++t) {
        if ((lane >> 3) == t) idreg = load_id(t);
    }
    auto issue = [&](uint64_t i) {
        const uint64_t g = i / nch;
        const uint32_t c0 = static_cast<uint32_t>(i % nch) * kChunk;
        const uint32_t cl = min(kChunk, a.d - c0);
        const uint32_t slot = (g % kIdAhead) * 8u;
        const uint64_t b = gbase(g);
        const uint32_t si = static_cast<uint32_t>(i % kStages);
        float* st = wr + si * kRows * kStride;
#pragma unroll
        for (uint32_t j = 0; j < kRows; ++j) {
            const uint32_t id = __shfl_sync(kFull, idreg, slot + j);
            if (b + j < mq && 4 * lane < cl) cp_async16(st + j * kStride + 4 * lane, a.data + uint64_t(id) * a.d + c0 + 4 * lane);
            if (lane == j) idbuf[warp][si][j] = id;
        }
        if (c0 + cl == a.d) {  // the group's last chunk is in flight: its id slots take group g + kIdAhead
            if ((lane >> 3) == g % kIdAhead) idreg = load_id(g + kIdAhead);
        }
    };
    double ld = kInf;
    uint32_t lid = 0xffffffffu;
    double acc = 0.0;
    float acc32 = 0.f;
    for (uint32_t i = 0; i + 1 < kStages; ++i) {
        if (i < items) issue(i);
        cp_async_commit();
    }
    for (uint64_t i = 0; i < items; ++i) {
        if (i + kStages - 1 < items) issue(i + kStages - 1);
        cp_async_commit();
        cp_async_wait<kStages - 1>();  // item i has landed (this lane's copies)
        __syncwarp();                  // ... and every lane's
        const uint64_t g = i / nch;
        const uint32_t c0 = static_cast<uint32_t>(i % nch) * kChunk;
        const uint32_t cl = min(kChunk, a.d - c0);
        const uint64_t b = gbase(g);
        const uint32_t nrows = static_cast<uint32_t>(min_u64(kRows, mq - b));
        if (r < nrows) {
            const float* row = wr + static_cast<uint32_t>(i % kStages) * kRows * kStride + r * kStride;
            if (use32) {
#pragma unroll 8
                for (uint32_t e = acc_i; e < cl; e += 4) {
                    const float df = row[e] - qf[c0 + e];
                    acc32 = __fmaf_rn(df, df, acc32);
                }
            } else {
#pragma unroll 8
                for (uint32_t e = acc_i; e < cl; e += 4) acc = __dadd_rn(acc, sqdiff_d(row[e], qd[c0 + e]));
            }
        }
        if (c0 + cl == a.d) {  // group done: combine the four chains, keep the top-k
            if (use32) acc = static_cast<double>(acc32);
            const double a1 = __shfl_down_sync(kFull, acc, 1);
            const double a2 = __shfl_down_sync(kFull, acc, 2);
            const double a3 = __shfl_down_sync(kFull, acc, 3);
            const double dist = __dadd_rn(__dadd_rn(acc, a1), __dadd_rn(a2, a3));  // valid on lanes 4r
            const uint32_t* ids = idbuf[warp][static_cast<uint32_t>(i % kStages)];
            acc = 0.0;
            acc32 = 0.f;
            if constexpr (GENERIC) {
                if (acc_i == 0 && r < nrows) {
                    a.all_d[q * a.m + b + r] = dist;
                    a.all_id[q * a.m + b + r] = ids[r];
                }
            } else {
#pragma unroll
                for (uint32_t j = 0; j < kRows; ++j) {
                    const double dj = __shfl_sync(kFull, dist, 4 * j);
                    if (j < nrows) warp_insert(dj, ids[j], ld, lid, a.k, lane);
                }
            }
        }
        __syncwarp();  // the slot (rows and ids) is refilled by the next iteration's issue
    }
    cp_async_wait<0>();
    if constexpr (!GENERIC) {
        __syncthreads();
        double* md = reinterpret_cast<double*>(ring);
        uint32_t* mi = reinterpret_cast<uint32_t*>(md + kWarps * 32);
        md[warp * 32 + lane] = ld;
        mi[warp * 32 + lane] = lid;
        __syncthreads();
        if (warp == 0) {
            for (uint32_t w = 1; w < kWarps; ++w) {
                for (uint32_t i = 0; i < a.k; ++i) {
                    const double dv = md[w * 32 + i];
                    if (dv == kInf) break;
                    warp_insert(dv, mi[w * 32 + i], ld, lid, a.k, lane);
                }
            }
            if (lane < a.k) {
                a.out_ids[q * a.k + lane] = lid;
                a.out_dists[q * a.k + lane] = a.squared ? ld : __dsqrt_rn(ld);
            }
        }
    }
}

// ------------------------------------------------------- screened f32 rows
// k <= 32, d % 4 == 0. The pipelined gathers of rerank_pipe_kernel feed an fp32 SCREEN instead of
// the fp64 chains: each lane folds its chain with FFMA (t = fl(x - q), acc = fl(acc + t*t)) and
// the four chains combine in fp32. With u = 2^-24 and n = d/4 terms per chain, the screened value
// s satisfies |s - D| <= G*D + E for the reference's fp64 value D, where G = (n + 8) * u * 1.01 and
// E = 1e-38 covers underflow (non-finite s: the row always passes). Every warp keeps the k smallest
// upper bounds s*(1+G)+E it has seen; tau, their largest, bounds the final k-th distance from
// above (k rows are known to lie below it), so a row whose lower bound s*(1-G)-E exceeds tau can
// never enter the top-k. Rows that pass are kept (id, lower bound) in a per-warp buffer; at the
// end the CTA merges the warps' bounds into one tau, and only buffered rows still below it get
// the exact fp64 4-accumulator distance (rerank_kernel's chains, bit-identical to the reference).
// About k + a few rows per query reach fp64. If a warp's buffer overflows (masses of exact ties),
// the query is re-ranked exactly from scratch.
constexpr uint32_t kSurvCap = 128;

__device__ __forceinline__ void list_insert_val(double v, double& sl, uint32_t k, uint32_t lane) {
    const bool before = lane < k && sl <= v;
    const uint32_t pos = __popc(__ballot_sync(kFull, before));
    const double up = __shfl_up_sync(kFull, sl, 1);
    if (lane > pos) sl = up;
    else if (lane == pos) sl = v;
}

__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

// Exact fp64 distances (the reference's 4 chains) of `count` rows id_at(0..count) into the warp's
// (dist, id) list; `st` is 8 x stride floats of warp-private staging.
template <class IdAt>
__device__ void exact_rows(const RerankArgs& a, float* st, uint32_t stride, const double* qd, uint64_t count,
                           IdAt id_at, double& ld, uint32_t& lid, uint32_t lane) {
    const uint32_t r = lane >> 2, acc_i = lane & 3u;
    for (uint64_t b = 0; b < count; b += kRows) {
        const uint32_t nrows = static_cast<uint32_t>(min_u64(kRows, count - b));
        const uint32_t my = lane < nrows ? id_at(b + lane) : 0u;
        uint32_t id[kRows];
#pragma unroll
        for (uint32_t j = 0; j < kRows; ++j) id[j] = __shfl_sync(kFull, my, j);
        double acc = 0.0;
        for (uint32_t c0 = 0; c0 < a.d; c0 += kChunk) {
            const uint32_t cl = min(kChunk, a.d - c0);
#pragma unroll
            for (uint32_t j = 0; j < kRows; ++j) {
                if (j < nrows && 4 * lane < cl)
                    *reinterpret_cast<float4*>(st + j * stride + 4 * lane) = ldg4(a.data + uint64_t(id[j]) * a.d + c0 + 4 * lane);
            }
            __syncwarp();
            if (r < nrows) {
                const float* row = st + r * stride;
                for (uint32_t e = acc_i; e < cl; e += 4) acc = __dadd_rn(acc, sqdiff_d(row[e], qd[c0 + e]));
            }
            __syncwarp();
        }
        const double a1 = __shfl_down_sync(kFull, acc, 1);
        const double a2 = __shfl_down_sync(kFull, acc, 2);
        const double a3 = __shfl_down_sync(kFull, acc, 3);
        const double dist = __dadd_rn(__dadd_rn(acc, a1), __dadd_rn(a2, a3));
#pragma unroll
        for (uint32_t j = 0; j < kRows; ++j) {
            const double dj = __shfl_sync(kFull, dist, 4 * j);
            if (j < nrows) warp_insert(dj, id[j], ld, lid, a.k, lane);
        }
    }
}

template <uint32_t S, uint32_t MINB>
__global__ void __launch_bounds__(kThreads, MINB) rerank_screen_kernel(RerankArgs a, uint32_t stride) {
    extern __shared__ __align__(16) unsigned char smem[];
    float* qf = reinterpret_cast<float*>(smem);                                                  // d
    double* qd = reinterpret_cast<double*>(smem + ((a.d * 4 + 15) / 16) * 16);                   // d
    float* ring = reinterpret_cast<float*>(smem + ((a.d * 4 + 15) / 16) * 16 + ((a.d * 8 + 15) / 16) * 16);
    __shared__ uint32_t idbuf[kWarps][S][kRows];
    __shared__ uint32_t sid[kWarps][kSurvCap];
    __shared__ float slo[kWarps][kSurvCap];
    __shared__ double md[kWarps * 32];
    __shared__ uint32_t mi[kWarps * 32];
    __shared__ double tau_cta;
    __shared__ int ovf;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    uint64_t q;
    if (!rerank_query(a, q)) return;
    const float* query = a.queries + q * a.d;
    if (tid == 0) ovf = 0;
    bool qu8 = true;
    for (uint32_t i = tid; i < a.d; i += kThreads) {
        const float v = query[i];
        qd[i] = static_cast<double>(v);
        qf[i] = v;
        qu8 &= is_u8(v);
    }
    if (a.data8 && __syncthreads_and(qu8)) return;  // rerank_u8_kernel owns this query
    __syncthreads();

    const double G = (static_cast<double>(a.d / 4) + 8.0) * 5.9604644775390625e-08 * 1.01;  // (n + 8) u, u = 2^-24
    const double E = 1e-38;
    float* wr = ring + warp * S * kRows * stride;
    const uint32_t r = lane >> 2, acc_i = lane & 3u;
    const uint32_t* cands = a.cands + q * a.m;
    const uint64_t mq = a.counts ? a.counts[q] : a.m;
    const uint32_t nch = (a.d + kChunk - 1) / kChunk;
    const uint64_t first = uint64_t(warp) * kRows;
    const uint64_t groups = mq > first ? (mq - first + kRows * kWarps - 1) / (kRows * kWarps) : 0;
    const uint64_t items = groups * nch;
    auto gbase = [&](uint64_t g) { return first + g * kRows * kWarps; };
    auto load_id = [&](uint64_t g) -> uint32_t {
        const uint64_t i = gbase(g) + (lane & 7u);
        if (g >= groups || i >= mq) return 0u;
        return a.identity ? static_cast<uint32_t>(i) : __ldcs(cands + i);
    };
    uint32_t idreg = 0;
#pragma unroll
    for (uint32_t t = 0; t < kIdAhead; ++t) {
        if ((lane >> 3) == t) idreg = load_id(t);
    }
    // issue / compute positions kept as counters (group, chunk, ring slot): no 64-bit div/mod
    uint32_t ig = 0, ic = 0, is = 0;
    auto issue_next = [&]() {
        const uint32_t c0 = ic * kChunk;
        const uint32_t cl = min(kChunk, a.d - c0);
        const uint32_t slot = (ig % kIdAhead) * 8u;
        float* st = wr + is * kRows * stride;
        uint32_t id[kRows];
#pragma unroll
        for (uint32_t j = 0; j < kRows; ++j) id[j] = __shfl_sync(kFull, idreg, slot + j);
        const uint32_t id8 = __shfl_sync(kFull, idreg, slot + (lane & 7u));
        if (4 * lane < cl) {  // rows past mq read row 0 (ids are 0 there): their results are ignored
#pragma unroll
            for (uint32_t j = 0; j < kRows; ++j)
                cp_async16(st + j * stride + 4 * lane, a.data + uint64_t(id[j]) * a.d + c0 + 4 * lane);
        }
        if (lane < kRows) idbuf[warp][is][lane] = id8;
        if (c0 + cl == a.d) {  // the group's last chunk is in flight: its id slots take group ig + kIdAhead
            if ((lane >> 3) == ig % kIdAhead) idreg = load_id(ig + kIdAhead);
            ++ig;
            ic = 0;
        } else {
            ++ic;
        }
        is = is + 1 == S ? 0u : is + 1;
    };
    double sl = kInf;  // screen list: the k smallest upper bounds (lane i = entry i)
    uint32_t nsurv = 0;
    bool overflow = false;
    float acc = 0.f;
    for (uint32_t i = 0; i + 1 < S; ++i) {
        if (i < items) issue_next();
        cp_async_commit();
    }
    uint32_t cg = 0, cc = 0, cs = 0;  // compute position
    for (uint64_t i = 0; i < items; ++i) {
        if (i + S - 1 < items) issue_next();
        cp_async_commit();
        cp_async_wait<S - 1>();
        __syncwarp();
        const uint32_t c0 = cc * kChunk;
        const uint32_t cl = min(kChunk, a.d - c0);
        const uint64_t b = gbase(cg);
        const uint32_t nrows = static_cast<uint32_t>(min_u64(kRows, mq - b));
        const uint32_t si = cs;
        if (r < nrows) {
            const float* row = wr + si * kRows * stride + r * stride;
#pragma unroll 8
            for (uint32_t e = acc_i; e < cl; e += 4) {
                const float t = row[e] - qf[c0 + e];
                acc = __fmaf_rn(t, t, acc);
            }
        }
        if (c0 + cl == a.d) {
            const float a1 = __shfl_down_sync(kFull, acc, 1);
            const float a2 = __shfl_down_sync(kFull, acc, 2);
            const float a3 = __shfl_down_sync(kFull, acc, 3);
            const float sv = __fadd_rn(__fadd_rn(acc, a1), __fadd_rn(a2, a3));  // valid on lanes 4r
            acc = 0.f;
            const bool valid = acc_i == 0 && r < nrows;
            const bool fin = isfinite(sv);
            const double sd = static_cast<double>(sv);
            const double lo = fin ? sd * (1.0 - G) - E : 0.0;
            const double up = fin ? sd * (1.0 + G) + E : kInf;
            // the k smallest upper bounds so far
            const double tau0 = __shfl_sync(kFull, sl, a.k - 1);  // (every lane: never inside a && chain)
            uint32_t bal = __ballot_sync(kFull, valid && up < tau0);
            while (bal) {
                const uint32_t src = __ffs(bal) - 1;
                bal &= bal - 1;
                const double v = __shfl_sync(kFull, up, src);
                if (v < __shfl_sync(kFull, sl, a.k - 1)) list_insert_val(v, sl, a.k, lane);
            }
            const double tau = __shfl_sync(kFull, sl, a.k - 1);
            const uint32_t pass = __ballot_sync(kFull, valid && lo <= tau);
            if (pass && !overflow) {
                const uint32_t cnt = __popc(pass);
                if (nsurv + cnt > kSurvCap) {  // drop buffered rows the tighter tau now excludes
                    uint32_t kept = 0;
                    for (uint32_t t0 = 0; t0 < nsurv; t0 += 32) {
                        const uint32_t t = t0 + lane;
                        const bool in = t < nsurv;
                        const uint32_t idv = in ? sid[warp][t] : 0u;
                        const float lv = in ? slo[warp][t] : 0.f;
                        const bool keep = in && static_cast<double>(lv) <= tau;
                        const uint32_t kb = __ballot_sync(kFull, keep);
                        __syncwarp();
                        if (keep) {
                            const uint32_t p = kept + __popc(kb & ((1u << lane) - 1u));
                            sid[warp][p] = idv;
                            slo[warp][p] = lv;
                        }
                        kept += __popc(kb);
                        __syncwarp();
                    }
                    nsurv = kept;
                }
                if (nsurv + cnt > kSurvCap) {
                    overflow = true;
                } else {
                    if ((pass >> lane) & 1u) {
                        const uint32_t p = nsurv + __popc(pass & ((1u << lane) - 1u));
                        sid[warp][p] = idbuf[warp][si][r];
                        slo[warp][p] = __double2float_rd(lo);
                    }
                    nsurv += cnt;
                }
            }
        }
        __syncwarp();  // the slot (rows and ids) is refilled by the next iteration's issue
        if (c0 + cl == a.d) {
            ++cg;
            cc = 0;
        } else {
            ++cc;
        }
        cs = cs + 1 == S ? 0u : cs + 1;
    }
    cp_async_wait<0>();
    // one tau for the CTA: the k smallest upper bounds over every warp
    if (overflow && lane == 0) atomicOr(&ovf, 1);
    md[warp * 32 + lane] = sl;
    __syncthreads();
    if (warp == 0) {
        for (uint32_t w = 1; w < kWarps; ++w) {
            for (uint32_t i = 0; i < a.k; ++i) {
                const double v = md[w * 32 + i];
                if (!(v < __shfl_sync(kFull, sl, a.k - 1))) break;  // lists are sorted
                list_insert_val(v, sl, a.k, lane);
            }
        }
        const double t = __shfl_sync(kFull, sl, a.k - 1);
        if (lane == 0) tau_cta = t;
    }
    __syncthreads();
    const double tau = tau_cta;
    double ld = kInf;
    uint32_t lid = 0xffffffffu;
    float* st = wr;  // the drained ring is staging now
    if (ovf) {  // exact re-rank of the whole query, the warps splitting the candidates
        const uint64_t per = (mq + kWarps - 1) / kWarps, lo = min_u64(mq, warp * per), hi = min_u64(mq, lo + per);
        exact_rows(a, st, stride, qd, hi - lo,
                   [&](uint64_t t) { return a.identity ? static_cast<uint32_t>(lo + t) : cands[lo + t]; }, ld, lid, lane);
    } else {
        uint32_t kept = 0;  // survivors: buffered rows whose lower bound is within the CTA's tau
        for (uint32_t t0 = 0; t0 < nsurv; t0 += 32) {
            const uint32_t t = t0 + lane;
            const bool in = t < nsurv;
            const uint32_t idv = in ? sid[warp][t] : 0u;
            const bool keep = in && static_cast<double>(slo[warp][t]) <= tau;
            const uint32_t kb = __ballot_sync(kFull, keep);
            __syncwarp();
            if (keep) sid[warp][kept + __popc(kb & ((1u << lane) - 1u))] = idv;
            kept += __popc(kb);
            __syncwarp();
        }
        exact_rows(a, st, stride, qd, kept, [&](uint64_t t) { return sid[warp][t]; }, ld, lid, lane);
    }
    __syncthreads();
    md[warp * 32 + lane] = ld;
    mi[warp * 32 + lane] = lid;
    __syncthreads();
    if (warp == 0) {
        for (uint32_t w = 1; w < kWarps; ++w) {
            for (uint32_t i = 0; i < a.k; ++i) {
                const double dv = md[w * 32 + i];
                if (dv == kInf) break;
                warp_insert(dv, mi[w * 32 + i], ld, lid, a.k, lane);
            }
        }
        if (lane < a.k) {
            a.out_ids[q * a.k + lane] = lid;
            a.out_dists[q * a.k + lane] = a.squared ? ld : __dsqrt_rn(ld);
        }
    }
}


// ------------------------------------------------------- int8-screened float rows
// Float rows (not u8-valued), d % 4 == 0, d <= 128: the screen reads an int8 copy of every row
// (a quarter of the f32 bytes) instead of the f32 row. Row x = s*a + e_x with a = rint(x / s) in
// [-127, 127], s = max|x| / 127; the query likewise q = t*b + e_q. With I = a.b (one IDP.4A per 4
// dims, exact int32) and ||x - q||^2 = |x|^2 + |q|^2 - 2 x.q,
//     |x.q - s t I| <= ||s a|| ||e_q|| + ||t b|| ||e_x|| + ||e_x|| ||e_q||          (Cauchy-Schwarz)
// so every candidate gets certified bounds lo <= D <= up of the reference's fp64 distance D; the
// per-row |x|^2, ||s a|| and ||e_x|| are stored beside the int8 row (rounded up where they bound),
// and a relative slack of 2^-20 covers every fp32 / fp64 rounding involved (the reference's own
// 4-chain sum is within ~1e-14 of the real value). The screen / survivor / exact-fp64 logic is
// rerank_screen_kernel's: the k smallest upper bounds give tau; rows with lo <= tau survive into
// a per-warp buffer; the CTA merges tau and re-ranks the survivors exactly from the f32 rows. A
// row or query whose bounds are not finite always survives; a full buffer re-ranks the query
// exactly from scratch.
constexpr uint32_t kQ8Stages = 2;
constexpr uint32_t kQ8Cap = 192;

// TMA bulk copies (sm_90+ async proxy) with mbarrier completion: a warp's ring slot is filled by
// one cp.async.bulk per row (the row's int8 words + bound terms, one 112-byte copy at d = 96)
// instead of seven 16-byte cp.async per row.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try(unsigned long long* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
    while (!mbar_try(bar, parity)) {
    }
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

template <uint32_t NW, bool TMA>
__global__ void __launch_bounds__(kThreads, 2) rerank_q8_kernel(RerankArgs a, uint32_t stride) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr uint32_t su = (NW + 1) | 1u;  // NW row words + 1 meta word, odd 16-byte stride
    double* qd = reinterpret_cast<double*>(smem);                                     // d
    const uint32_t per_warp = max(kQ8Stages * 32 * su * 16, kRows * stride * 4);      // ring / staging
    unsigned char* wbase = smem + ((a.d * 8 + 15) / 16) * 16;
    __shared__ uint32_t qpack[32];
    __shared__ uint32_t sid[kWarps][kQ8Cap];
    __shared__ float slo[kWarps][kQ8Cap];
    __shared__ double md[kWarps * 32];
    __shared__ uint32_t mi[kWarps * 32];
    __shared__ double qpar[4];  // t, |q|^2, ||t b|| (up), ||e_q|| (up)
    __shared__ double tau_cta;
    __shared__ int ovf, qok;
    __shared__ __align__(8) unsigned long long mbar[kWarps][kQ8Stages];  // TMA: one per ring slot
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    uint64_t q;
    if (!rerank_query(a, q)) return;
    const float* query = a.queries + q * a.d;
    if constexpr (TMA) {
        if (lane < kQ8Stages) mbar_init(&mbar[warp][lane], 1);
        mbar_fence_init();
    }
    for (uint32_t i = tid; i < a.d; i += kThreads) qd[i] = static_cast<double>(query[i]);
    if (warp == 0) {  // quantise the query (d <= 128: lane owns dims 4 lane .. 4 lane + 3)
        float v[4], mx = 0.f;
#pragma unroll
        for (uint32_t j = 0; j < 4; ++j) {
            const uint32_t i = 4 * lane + j;
            v[j] = i < a.d ? query[i] : 0.f;
            mx = fmaxf(mx, fabsf(v[j]));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, o));
        const float t = mx / 127.f;
        double e2 = 0.0, b2 = 0.0, n2 = 0.0;
        uint32_t packed = 0;
#pragma unroll
        for (uint32_t j = 0; j < 4; ++j) {
            const float bq = t > 0.f ? fminf(127.f, fmaxf(-127.f, rintf(v[j] / t))) : 0.f;
            const double e = static_cast<double>(v[j]) - static_cast<double>(t) * static_cast<double>(bq);
            e2 += e * e;
            b2 += static_cast<double>(bq) * static_cast<double>(bq);
            n2 += static_cast<double>(v[j]) * static_cast<double>(v[j]);
            packed |= (static_cast<uint32_t>(static_cast<int>(bq)) & 0xffu) << (8 * j);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            e2 += __shfl_xor_sync(kFull, e2, o);
            b2 += __shfl_xor_sync(kFull, b2, o);
            n2 += __shfl_xor_sync(kFull, n2, o);
        }
        qpack[lane] = packed;
        if (lane == 0) {
            qpar[0] = static_cast<double>(t);
            qpar[1] = n2;
            qpar[2] = static_cast<double>(t) * sqrt(b2) * (1.0 + 1e-12);
            qpar[3] = sqrt(e2) * (1.0 + 1e-12);
            qok = isfinite(n2) && isfinite(e2) && isfinite(qpar[2]);
            ovf = 0;
        }
    }
    __syncthreads();
    int qv[NW][4];
#pragma unroll
    for (uint32_t w = 0; w < NW; ++w) {
#pragma unroll
        for (uint32_t j = 0; j < 4; ++j) qv[w][j] = static_cast<int>(qpack[4 * w + j]);
    }
    const double qt = qpar[0], n2q = qpar[1], Bq = qpar[2], rq = qpar[3];
    const bool qfin = qok != 0;
    uint4* ring = reinterpret_cast<uint4*>(wbase + warp * per_warp);
    const uint32_t* cands = a.cands + q * a.m;
    const uint64_t mq = a.counts ? a.counts[q] : a.m;
    const uint64_t first = uint64_t(warp) * 32;
    const uint64_t steps = mq > first ? (mq - first + 32 * kWarps - 1) / (32 * kWarps) : 0;
    auto sbase = [&](uint64_t g) { return first + g * 32 * kWarps; };
    auto load_id = [&](uint64_t g) -> uint32_t {
        const uint64_t i = sbase(g) + lane;
        if (g >= steps || i >= mq) return 0u;
        return a.identity ? static_cast<uint32_t>(i) : __ldcs(cands + i);
    };
    uint32_t id0 = load_id(0), id1 = load_id(1);
    auto issue = [&](uint64_t g) {
        const uint32_t myid = (g & 1u) ? id1 : id0;
        const uint32_t slot = static_cast<uint32_t>(g % kQ8Stages);
        uint4* st = ring + slot * 32 * su;
        const uint64_t b = sbase(g);
        if constexpr (TMA) {
            const uint32_t nvalid = static_cast<uint32_t>(min_u64(32, mq - b));
            fence_proxy_async();  // the slot's previous contents were read by the generic proxy
            __syncwarp();
            if (lane == 0) mbar_expect_tx(&mbar[warp][slot], nvalid * (NW + 1) * 16u);
            __syncwarp();
            if (lane < nvalid) bulk_g2s(st + lane * su, a.q8 + uint64_t(myid) * a.qrec, (NW + 1) * 16u, &mbar[warp][slot]);
        } else {
#pragma unroll
            for (uint32_t t = lane; t < 32 * (NW + 1); t += 32) {
                const uint32_t row = t / (NW + 1), col = t % (NW + 1);
                const uint32_t id = __shfl_sync(kFull, myid, row);
                if (b + row < mq) cp_async16(st + row * su + col, a.q8 + uint64_t(id) * a.qrec + 16u * col);
            }
        }
        if (g & 1u) id1 = load_id(g + 2);
        else id0 = load_id(g + 2);
        return myid;
    };
    uint32_t rowid[kQ8Stages];
#pragma unroll
    for (uint32_t i = 0; i < kQ8Stages; ++i) rowid[i] = 0;
    if constexpr (TMA) __syncwarp();  // the barriers are initialised
    for (uint32_t i = 0; i + 1 < kQ8Stages; ++i) {
        if (i < steps) rowid[i] = issue(i);
        if constexpr (!TMA) cp_async_commit();
    }
    double sl = kInf;  // the k smallest upper bounds (lane i = entry i)
    uint32_t nsurv = 0;
    bool overflow = false;
    for (uint64_t g = 0; g < steps; ++g) {
        if (g + kQ8Stages - 1 < steps) {
            const uint32_t v = issue(g + kQ8Stages - 1);
            const uint32_t slot = static_cast<uint32_t>((g + kQ8Stages - 1) % kQ8Stages);
#pragma unroll
            for (uint32_t i = 0; i < kQ8Stages; ++i) {
                if (i == slot) rowid[i] = v;
            }
        }
        if constexpr (TMA) {
            mbar_wait(&mbar[warp][g % kQ8Stages], static_cast<uint32_t>((g / kQ8Stages) & 1u));
        } else {
            cp_async_commit();
            cp_async_wait<kQ8Stages - 1>();
        }
        __syncwarp();
        const uint32_t slot = static_cast<uint32_t>(g % kQ8Stages);
        uint32_t myid = rowid[0];
#pragma unroll
        for (uint32_t i = 1; i < kQ8Stages; ++i) {
            if (i == slot) myid = rowid[i];
        }
        const uint4* row = ring + slot * 32 * su + lane * su;
        int c0 = 0, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
        for (uint32_t w = 0; w < NW; ++w) {
            const uint4 x = row[w];
            c0 = __dp4a(static_cast<int>(x.x), qv[w][0], c0);
            c1 = __dp4a(static_cast<int>(x.y), qv[w][1], c1);
            c2 = __dp4a(static_cast<int>(x.z), qv[w][2], c2);
            c3 = __dp4a(static_cast<int>(x.w), qv[w][3], c3);
        }
        const uint4 mw = row[NW];
        __syncwarp();  // the slot is refilled by the next step's issue
        const int I = (c0 + c1) + (c2 + c3);
        const float rs = __uint_as_float(mw.x), rn2 = __uint_as_float(mw.y);
        const float rA = __uint_as_float(mw.z), rR = __uint_as_float(mw.w);
        const uint64_t b = sbase(g);
        const bool valid = b + lane < mq;
        double lo = 0.0, up = kInf;
        if (qfin && rs >= 0.f) {
            const double dot = static_cast<double>(rs) * qt * static_cast<double>(I);
            const double approx = static_cast<double>(rn2) + n2q - 2.0 * dot;
            const double err = 2.0 * (static_cast<double>(rA) * rq + Bq * static_cast<double>(rR) +
                                      static_cast<double>(rR) * rq);
            const double slack = 9.5367431640625e-07 * (static_cast<double>(rn2) + n2q + 2.0 * fabs(dot)) + 1e-300;
            lo = approx - err - slack;
            up = approx + err + slack;
        }
        const double tau0 = __shfl_sync(kFull, sl, a.k - 1);
        uint32_t bal = __ballot_sync(kFull, valid && up < tau0);
        while (bal) {
            const uint32_t src = __ffs(bal) - 1;
            bal &= bal - 1;
            const double v = __shfl_sync(kFull, up, src);
            if (v < __shfl_sync(kFull, sl, a.k - 1)) list_insert_val(v, sl, a.k, lane);
        }
        const double tau = __shfl_sync(kFull, sl, a.k - 1);
        const uint32_t pass = __ballot_sync(kFull, valid && lo <= tau);
        if (pass && !overflow) {
            const uint32_t cnt = __popc(pass);
            if (nsurv + cnt > kQ8Cap) {  // drop buffered rows the tighter tau now excludes
                uint32_t kept = 0;
                for (uint32_t t0 = 0; t0 < nsurv; t0 += 32) {
                    const uint32_t t = t0 + lane;
                    const bool in = t < nsurv;
                    const uint32_t idv = in ? sid[warp][t] : 0u;
                    const float lv = in ? slo[warp][t] : 0.f;
                    const bool keep = in && static_cast<double>(lv) <= tau;
                    const uint32_t kb = __ballot_sync(kFull, keep);
                    __syncwarp();
                    if (keep) {
                        const uint32_t p = kept + __popc(kb & ((1u << lane) - 1u));
                        sid[warp][p] = idv;
                        slo[warp][p] = lv;
                    }
                    kept += __popc(kb);
                    __syncwarp();
                }
                nsurv = kept;
            }
            if (nsurv + cnt > kQ8Cap) {
                overflow = true;
            } else {
                if ((pass >> lane) & 1u) {
                    const uint32_t p = nsurv + __popc(pass & ((1u << lane) - 1u));
                    sid[warp][p] = myid;
                    slo[warp][p] = __double2float_rd(lo);
                }
                nsurv += cnt;
            }
            __syncwarp();
        }
    }
    if constexpr (!TMA) cp_async_wait<0>();  // (TMA: every issued slot was waited on in the loop)
    if (overflow && lane == 0) atomicOr(&ovf, 1);
    md[warp * 32 + lane] = sl;
    __syncthreads();
    if (warp == 0) {
        for (uint32_t w = 1; w < kWarps; ++w) {
            for (uint32_t i = 0; i < a.k; ++i) {
                const double v = md[w * 32 + i];
                if (!(v < __shfl_sync(kFull, sl, a.k - 1))) break;  // lists are sorted
                list_insert_val(v, sl, a.k, lane);
            }
        }
        const double t = __shfl_sync(kFull, sl, a.k - 1);
        if (lane == 0) tau_cta = t;
    }
    __syncthreads();
    const double tau = tau_cta;
    double ld = kInf;
    uint32_t lid = 0xffffffffu;
    float* st = reinterpret_cast<float*>(ring);  // the drained ring is staging now
    if (ovf) {  // exact re-rank of the whole query, the warps splitting the candidates
        const uint64_t per = (mq + kWarps - 1) / kWarps, lo = min_u64(mq, warp * per), hi = min_u64(mq, lo + per);
        if (a.screen_stats && tid == 0) atomicAdd(a.screen_stats + 1, 1ull);
        exact_rows(a, st, stride, qd, hi - lo,
                   [&](uint64_t t) { return a.identity ? static_cast<uint32_t>(lo + t) : cands[lo + t]; }, ld, lid, lane);
    } else {
        uint32_t kept = 0;  // survivors: buffered rows whose lower bound is within the CTA's tau
        for (uint32_t t0 = 0; t0 < nsurv; t0 += 32) {
            const uint32_t t = t0 + lane;
            const bool in = t < nsurv;
            const uint32_t idv = in ? sid[warp][t] : 0u;
            const bool keep = in && static_cast<double>(slo[warp][t]) <= tau;
            const uint32_t kb = __ballot_sync(kFull, keep);
            __syncwarp();
            if (keep) sid[warp][kept + __popc(kb & ((1u << lane) - 1u))] = idv;
            kept += __popc(kb);
            __syncwarp();
        }
        if (a.screen_stats && lane == 0) atomicAdd(a.screen_stats, static_cast<unsigned long long>(kept));
        exact_rows(a, st, stride, qd, kept, [&](uint64_t t) { return sid[warp][t]; }, ld, lid, lane);
    }
    __syncthreads();
    md[warp * 32 + lane] = ld;
    mi[warp * 32 + lane] = lid;
    __syncthreads();
    if (warp == 0) {
        for (uint32_t w = 1; w < kWarps; ++w) {
            for (uint32_t i = 0; i < a.k; ++i) {
                const double dv = md[w * 32 + i];
                if (dv == kInf) break;
                warp_insert(dv, mi[w * 32 + i], ld, lid, a.k, lane);
            }
        }
        if (lane < a.k) {
            a.out_ids[q * a.k + lane] = lid;
            a.out_dists[q * a.k + lane] = a.squared ? ld : __dsqrt_rn(ld);
        }
    }
}

// ------------------------------------------- int8 screen with a prefix bound (NW >= 4)
// Record (qrec bytes, a multiple of 64) in two arrays: [meta0][dims 0 .. 16 kQ8P) — qsplit bytes (32
// for one prefix word, 64 for three), the n prefix parts back to back at q8 — and
// [dims 16 kQ8P .. 16 NW)[meta1] at q8b, stride qrec - qsplit; meta0 = (s, |a_S|^2
// (u32 bits), ||e_x,S|| up, 0), meta1 = (|a|^2 (u32 bits), ||e_x|| up, s, 0), S = the prefix dims.
// Stage 1 reads the prefix part of every candidate. The prefix alone bounds the distance from below:
//     D >= sum_{i in S} (x_i - q_i)^2 >= (||s a_S - t b_S|| - ||e_x,S|| - ||e_q,S||)^2,
//     ||s a_S - t b_S||^2 = s^2 |a_S|^2 + t^2 |b_S|^2 - 2 s t (a_S . b_S),   a_S . b_S exact (IDP.4A)
// (at cfg4 the first 24 of 96 dims rule out about 98 % of the candidates against the final k-th
// distance, tools/partial_bound.py; the compaction puts score > T candidates first, so tau is
// close to final early). Rows still under tau queue (id, a_S . b_S); 32 queued rows
// make one stage-2 batch, whose rest-of-row words and meta1 give rerank_q8_kernel's full
// certified bounds (tau, exact survivors). A batch is issued in the same cp.async group as the
// next prefix step and consumed one step later, so the copies never drain; tau is shared across
// the CTA's warps (the minimum of their k-th upper bounds bounds the query's k-th distance).
constexpr uint32_t kQ8QCap = 64;  // queued rows per warp (at most 63 by construction)

// Certified bounds lo <= D <= up of the reference's fp64 squared distance from the int8 forms
// x = s a + e_x, q = t b + e_q: ||x - q|| is within ||e_x|| + ||e_q|| of ||s a - t b||, whose square
// s^2 |a|^2 + t^2 |b|^2 - 2 s t (a . b) is exact up to fp64 rounding (a . b exact from IDP.4A). The
// error is relative to sqrt(D), not to |x| (the Cauchy-Schwarz form |x.q - s t a.b| <= ... is not:
// at cfg3, rows of norm 17 at distance 2, it let a thousand candidates per query through).
__device__ __forceinline__ void tri_bounds(double s, double a2, double tb2, double qt, int I, double ex, double eq,
                                           double& lo, double& up) {
    const double sa = s * s * a2;
    const double cr = 2.0 * s * qt * static_cast<double>(I);
    const double V = sa + tb2 - cr;
    const double sl = 1.1368683772161603e-13 * (sa + tb2 + fabs(cr));  // 2^-43: every fp64 rounding above
    const double rlo = sqrt(fmax(V - sl, 0.0)) * (1.0 - 1e-15) - ex - eq;
    const double rhi = sqrt(fmax(V + sl, 0.0)) * (1.0 + 1e-15) + ex + eq;
    lo = rlo > 0.0 ? rlo * rlo * (1.0 - 1e-9) : 0.0;  // (1e-9: the reference's 4-chain sum vs the real value)
    up = rhi * rhi * (1.0 + 1e-9);
}

// Stage 1 of the prefix screens without a square root per row. The prefix bound is lb = r^2 (1 - 1e-9)
// with r = sqrt(max(V, 0)) (1 - 1e-15) - e_S - e_qS (0 when r <= 0), and a row is queued when
// lb <= tau. Every such row satisfies sqrt(V) (1 - 2e-15) <= rt + e_S + e_qS with
// rt = sqrt(tau (1 + 3e-9)) (1 + 1e-15), i.e. V (1 - 4e-14) <= (rt + e_S + e_qS)^2 with room for the
// roundings on both sides: the test below keeps a superset of the rows the bound keeps, so it is as
// certified as the bound, and the square root is taken once per change of tau instead of per row.
struct PrefixGate {
    double tau = -1.0, rtq = kInf;  // the tau the gate was built for; rt + e_qS
    __device__ __forceinline__ void update(double tau_new, double eqS) {
        if (tau_new != tau) {
            tau = tau_new;
            rtq = tau_new < kInf ? sqrt(tau_new * (1.0 + 3e-9)) * (1.0 + 1e-15) + eqS : kInf;
        }
    }
    __device__ __forceinline__ bool keeps(double V, float eS) const {
        const double c = rtq + static_cast<double>(eS);
        return !(fmax(V, 0.0) * (1.0 - 4e-14) > c * c);  // (NaN: kept, as the bound's lb = 0 is)
    }
};

template <uint32_t kQ8P, uint32_t NR>  // prefix words (16 dims each), rest words: NW = kQ8P + NR
__global__ void __launch_bounds__(kThreads, 2) rerank_q8p_kernel(RerankArgs a, uint32_t stride) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr uint32_t NW = kQ8P + NR;
    constexpr uint32_t suA = (kQ8P + 1) | 1u;  // meta0 + prefix words, odd 16-byte stride
    constexpr uint32_t suB = (NR + 1) | 1u;  // NR words + meta1, odd stride
    double* qd = reinterpret_cast<double*>(smem);  // d
    const uint32_t ringA = kQ8Stages * 32 * suA, ringB = 2 * 32 * suB;  // uint4 units
    const uint32_t per_warp = max((ringA + ringB) * 16, kRows * stride * 4);
    unsigned char* wbase = smem + ((a.d * 8 + 15) / 16) * 16;
    __shared__ uint32_t qpack[32];
    __shared__ uint32_t sid[kWarps][kQ8Cap];
    __shared__ float slo[kWarps][kQ8Cap];
    __shared__ uint32_t qqid[kWarps][kQ8QCap];
    __shared__ int qqI[kWarps][kQ8QCap];
    __shared__ double md[kWarps * 32];
    __shared__ uint32_t mi[kWarps * 32];
    __shared__ double qpar[7];  // t, |q|^2, ||t b|| (up), ||e_q|| (up), t^2 |b_S|^2, ||e_q,S|| (up), t^2 |b|^2
    __shared__ double tau_cta;
    __shared__ unsigned long long tau_sh;  // CTA-wide min of the warps' k-th upper bounds (bits of a double >= 0)
    __shared__ int ovf, qok;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    uint64_t q;
    if (!rerank_query(a, q)) return;
    const float* query = a.queries + q * a.d;
    for (uint32_t i = tid; i < a.d; i += kThreads) qd[i] = static_cast<double>(query[i]);
    if (warp == 0) {  // quantise the query (d <= 128: lane owns dims 4 lane .. 4 lane + 3)
        float v[4], mx = 0.f;
#pragma unroll
        for (uint32_t j = 0; j < 4; ++j) {
            const uint32_t i = 4 * lane + j;
            v[j] = i < a.d ? query[i] : 0.f;
            mx = fmaxf(mx, fabsf(v[j]));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, o));
        const float t = mx / 127.f;
        double e2 = 0.0, b2 = 0.0, n2 = 0.0;
        uint32_t packed = 0;
#pragma unroll
        for (uint32_t j = 0; j < 4; ++j) {
            const float bq = t > 0.f ? fminf(127.f, fmaxf(-127.f, rintf(v[j] / t))) : 0.f;
            const double e = static_cast<double>(v[j]) - static_cast<double>(t) * static_cast<double>(bq);
            e2 += e * e;
            b2 += static_cast<double>(bq) * static_cast<double>(bq);
            n2 += static_cast<double>(v[j]) * static_cast<double>(v[j]);
            packed |= (static_cast<uint32_t>(static_cast<int>(bq)) & 0xffu) << (8 * j);
        }
        const bool pre = lane < 4 * kQ8P;  // this lane's dims are in the prefix
        double e2s = pre ? e2 : 0.0, b2s = pre ? b2 : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            e2 += __shfl_xor_sync(kFull, e2, o);
            b2 += __shfl_xor_sync(kFull, b2, o);
            n2 += __shfl_xor_sync(kFull, n2, o);
            e2s += __shfl_xor_sync(kFull, e2s, o);
            b2s += __shfl_xor_sync(kFull, b2s, o);
        }
        qpack[lane] = packed;
        if (lane == 0) {
            qpar[0] = static_cast<double>(t);
            qpar[1] = n2;
            qpar[2] = static_cast<double>(t) * sqrt(b2) * (1.0 + 1e-12);
            qpar[3] = sqrt(e2) * (1.0 + 1e-12);
            qpar[4] = static_cast<double>(t) * static_cast<double>(t) * b2s;  // b2s: an exact integer
            qpar[5] = sqrt(e2s) * (1.0 + 1e-12);
            qpar[6] = static_cast<double>(t) * static_cast<double>(t) * b2;
            qok = isfinite(n2) && isfinite(e2) && isfinite(qpar[2]);
            ovf = 0;
            tau_sh = 0x7ff0000000000000ull;  // +inf
        }
    }
    __syncthreads();
    int qv[NW][4];
#pragma unroll
    for (uint32_t w = 0; w < NW; ++w) {
#pragma unroll
        for (uint32_t j = 0; j < 4; ++j) qv[w][j] = static_cast<int>(qpack[4 * w + j]);
    }
    const double qt = qpar[0], rq = qpar[3], tb2S = qpar[4], eqS = qpar[5], tb2 = qpar[6];
    const bool qfin = qok != 0;
    uint4* ra = reinterpret_cast<uint4*>(wbase + warp * per_warp);
    uint4* rb = ra + ringA;
    uint32_t* qid = qqid[warp];
    int* qI = qqI[warp];
    const uint32_t* cands = a.cands + q * a.m;
    const uint64_t mq = a.counts ? a.counts[q] : a.m;
    const uint64_t first = uint64_t(warp) * 32;
    const uint64_t steps = mq > first ? (mq - first + 32 * kWarps - 1) / (32 * kWarps) : 0;
    auto sbase = [&](uint64_t g) { return first + g * 32 * kWarps; };
    auto load_id = [&](uint64_t g) -> uint32_t {
        const uint64_t i = sbase(g) + lane;
        if (g >= steps || i >= mq) return 0u;
        return a.identity ? static_cast<uint32_t>(i) : __ldcs(cands + i);
    };
    uint32_t id0 = load_id(0), id1 = load_id(1);
    auto issue_a = [&](uint64_t g) {  // granule 0 of the step's 32 rows
        const uint32_t myid = (g & 1u) ? id1 : id0;
        uint4* st = ra + static_cast<uint32_t>(g % kQ8Stages) * 32 * suA;
        const uint64_t b = sbase(g);
#pragma unroll
        for (uint32_t t = lane; t < 32 * (kQ8P + 1); t += 32) {
            const uint32_t row = t / (kQ8P + 1), col = t % (kQ8P + 1);
            const uint32_t id = __shfl_sync(kFull, myid, row);
            if (b + row < mq) cp_async16(st + row * suA + col, a.q8 + uint64_t(id) * a.qsplit + 16u * col);
        }
        if (g & 1u) id1 = load_id(g + 2);
        else id0 = load_id(g + 2);
        return myid;
    };
    auto issue_b = [&](uint32_t slot, uint32_t cnt, uint32_t bid) {  // the rest of the batch's rows
        uint4* st = rb + slot * 32 * suB;
#pragma unroll
        for (uint32_t t = lane; t < 32 * (NR + 1); t += 32) {
            const uint32_t row = t / (NR + 1), col = t % (NR + 1);
            const uint32_t id = __shfl_sync(kFull, bid, row);
            if (row < cnt) cp_async16(st + row * suB + col, a.q8b + uint64_t(id) * (a.qrec - a.qsplit) + 16u * col);
        }
    };
    uint32_t rowid0 = 0, rowid1 = 0;
    if (steps) rowid0 = issue_a(0);
    cp_async_commit();
    double sl = kInf;  // this warp's k smallest upper bounds (lane i = entry i)
    uint32_t nsurv = 0, qn = 0;
    bool overflow = false;
    uint32_t fcnt = 0, fid = 0, fslot = 0, nslot = 0;  // the batch in flight (issued last iteration)
    int fI = 0;
    auto tau_now = [&]() {
        const double own = __shfl_sync(kFull, sl, a.k - 1);
        const double shared = __longlong_as_double(static_cast<long long>(*reinterpret_cast<volatile unsigned long long*>(&tau_sh)));
        return fmin(own, shared);
    };
    PrefixGate gate;
    for (uint64_t g = 0; g < steps || fcnt || qn; ++g) {
        if (g + 1 < steps) {
            const uint32_t v = issue_a(g + 1);
            if (g & 1u) rowid0 = v;
            else rowid1 = v;
        }
        // a new batch: 32 queued rows, or whatever is left once the prefix steps are done
        uint32_t ncnt = 0, nid = 0;
        int nI = 0;
        if (qn >= 32 || (g >= steps && qn)) {
            ncnt = min(qn, 32u);
            if (lane < ncnt) {
                nid = qid[lane];
                nI = qI[lane];
            }
            const uint32_t r0 = 32 + lane < qn ? qid[32 + lane] : 0u;  // the rest moves to the front
            const int r1 = 32 + lane < qn ? qI[32 + lane] : 0;
            __syncwarp();
            if (32 + lane < qn) {
                qid[lane] = r0;
                qI[lane] = r1;
            }
            __syncwarp();
            qn -= ncnt;
            issue_b(nslot, ncnt, nid);
        }
        cp_async_commit();
        cp_async_wait<1>();  // the prefix step g and the batch issued last iteration have landed
        __syncwarp();
        if (fcnt) {  // stage 2: full certified bounds of the batch
            if (a.screen_stats && lane == 0) atomicAdd(a.screen_stats + 2, static_cast<unsigned long long>(fcnt));
            const uint4* row = rb + fslot * 32 * suB + lane * suB;
            int c0 = fI, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
            for (uint32_t w = 0; w < NR; ++w) {
                const uint4 x = row[w];
                c0 = __dp4a(static_cast<int>(x.x), qv[kQ8P + w][0], c0);
                c1 = __dp4a(static_cast<int>(x.y), qv[kQ8P + w][1], c1);
                c2 = __dp4a(static_cast<int>(x.z), qv[kQ8P + w][2], c2);
                c3 = __dp4a(static_cast<int>(x.w), qv[kQ8P + w][3], c3);
            }
            const uint4 mw = row[NR];  // meta1 = (|a|^2, ||e_x|| up, s, 0)
            const int I = (c0 + c1) + (c2 + c3);
            const float rR = __uint_as_float(mw.y), rs = __uint_as_float(mw.z);
            const bool valid = lane < fcnt;
            double lo = 0.0, up = kInf;
            if (qfin && rs >= 0.f)
                tri_bounds(static_cast<double>(rs), static_cast<double>(mw.x), tb2, qt, I, static_cast<double>(rR), rq, lo, up);
            const double tau0 = __shfl_sync(kFull, sl, a.k - 1);
            uint32_t bal = __ballot_sync(kFull, valid && up < tau0);
            if (bal) {
                while (bal) {
                    const uint32_t src = __ffs(bal) - 1;
                    bal &= bal - 1;
                    const double v = __shfl_sync(kFull, up, src);
                    if (v < __shfl_sync(kFull, sl, a.k - 1)) list_insert_val(v, sl, a.k, lane);
                }
                const double own = __shfl_sync(kFull, sl, a.k - 1);
                if (lane == 0 && own < kInf && own >= 0.0)
                    atomicMin(&tau_sh, static_cast<unsigned long long>(__double_as_longlong(own)));
            }
            const double tau = tau_now();
            const uint32_t pass = __ballot_sync(kFull, valid && lo <= tau);
            if (pass && !overflow) {
                const uint32_t cnt = __popc(pass);
                if (nsurv + cnt > kQ8Cap) {  // drop buffered rows the tighter tau now excludes
                    uint32_t kept = 0;
                    for (uint32_t t0 = 0; t0 < nsurv; t0 += 32) {
                        const uint32_t t = t0 + lane;
                        const bool in = t < nsurv;
                        const uint32_t idv = in ? sid[warp][t] : 0u;
                        const float lv = in ? slo[warp][t] : 0.f;
                        const bool keep = in && static_cast<double>(lv) <= tau;
                        const uint32_t kb = __ballot_sync(kFull, keep);
                        __syncwarp();
                        if (keep) {
                            const uint32_t p = kept + __popc(kb & ((1u << lane) - 1u));
                            sid[warp][p] = idv;
                            slo[warp][p] = lv;
                        }
                        kept += __popc(kb);
                        __syncwarp();
                    }
                    nsurv = kept;
                }
                if (nsurv + cnt > kQ8Cap) {
                    overflow = true;
                } else {
                    if ((pass >> lane) & 1u) {
                        const uint32_t p = nsurv + __popc(pass & ((1u << lane) - 1u));
                        sid[warp][p] = fid;
                        slo[warp][p] = __double2float_rd(lo);
                    }
                    nsurv += cnt;
                }
                __syncwarp();
            }
        }
        fcnt = ncnt;
        fid = nid;
        fI = nI;
        fslot = nslot;
        nslot ^= 1u;
        if (g < steps) {  // stage 1: the prefix bound of step g's rows
            const uint32_t myid = (g & 1u) ? rowid1 : rowid0;
            const uint4* row = ra + static_cast<uint32_t>(g % kQ8Stages) * 32 * suA + lane * suA;
            const uint4 m0 = row[0];
            int c0 = 0, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
            for (uint32_t w = 0; w < kQ8P; ++w) {
                const uint4 x = row[1 + w];
                c0 = __dp4a(static_cast<int>(x.x), qv[w][0], c0);
                c1 = __dp4a(static_cast<int>(x.y), qv[w][1], c1);
                c2 = __dp4a(static_cast<int>(x.z), qv[w][2], c2);
                c3 = __dp4a(static_cast<int>(x.w), qv[w][3], c3);
            }
            __syncwarp();  // the slot is refilled by the next issue
            const int IS = (c0 + c1) + (c2 + c3);
            const float rs = __uint_as_float(m0.x), eS = __uint_as_float(m0.z);
            const bool valid = sbase(g) + lane < mq;
            gate.update(tau_now(), eqS);
            bool under = true;  // the prefix bound is within tau (PrefixGate: no square root per row)
            if (qfin && rs >= 0.f) {
                const double s = static_cast<double>(rs);
                const double sa = s * s * static_cast<double>(m0.y);  // |a_S|^2: an exact integer
                const double cr = 2.0 * s * qt * static_cast<double>(IS);
                const double V = sa + tb2S - cr - 1.1368683772161603e-13 * (sa + tb2S + fabs(cr));  // 2^-43 slack
                under = gate.keeps(V, eS);
            }
            const uint32_t keep = __ballot_sync(kFull, valid && under);
            if (keep) {
                if ((keep >> lane) & 1u) {
                    const uint32_t p = qn + __popc(keep & ((1u << lane) - 1u));
                    qid[p] = myid;
                    qI[p] = IS;
                }
                qn += __popc(keep);
                __syncwarp();
            }
        }
    }
    cp_async_wait<0>();
    if (overflow && lane == 0) atomicOr(&ovf, 1);
    md[warp * 32 + lane] = sl;
    __syncthreads();
    if (warp == 0) {
        for (uint32_t w = 1; w < kWarps; ++w) {
            for (uint32_t i = 0; i < a.k; ++i) {
                const double v = md[w * 32 + i];
                if (!(v < __shfl_sync(kFull, sl, a.k - 1))) break;  // lists are sorted
                list_insert_val(v, sl, a.k, lane);
            }
        }
        const double t = __shfl_sync(kFull, sl, a.k - 1);
        if (lane == 0) tau_cta = t;
    }
    __syncthreads();
    const double tau = tau_cta;
    double ld = kInf;
    uint32_t lid = 0xffffffffu;
    float* st = reinterpret_cast<float*>(ra);  // the drained rings are staging now
    if (ovf) {  // exact re-rank of the whole query, the warps splitting the candidates
        const uint64_t per = (mq + kWarps - 1) / kWarps, lo = min_u64(mq, warp * per), hi = min_u64(mq, lo + per);
        if (a.screen_stats && tid == 0) atomicAdd(a.screen_stats + 1, 1ull);
        exact_rows(a, st, stride, qd, hi - lo,
                   [&](uint64_t t) { return a.identity ? static_cast<uint32_t>(lo + t) : cands[lo + t]; }, ld, lid, lane);
    } else {
        uint32_t kept = 0;  // survivors: buffered rows whose lower bound is within the CTA's tau
        for (uint32_t t0 = 0; t0 < nsurv; t0 += 32) {
            const uint32_t t = t0 + lane;
            const bool in = t < nsurv;
            const uint32_t idv = in ? sid[warp][t] : 0u;
            const bool keep = in && static_cast<double>(slo[warp][t]) <= tau;
            const uint32_t kb = __ballot_sync(kFull, keep);
            __syncwarp();
            if (keep) sid[warp][kept + __popc(kb & ((1u << lane) - 1u))] = idv;
            kept += __popc(kb);
            __syncwarp();
        }
        if (a.screen_stats && lane == 0) atomicAdd(a.screen_stats, static_cast<unsigned long long>(kept));
        exact_rows(a, st, stride, qd, kept, [&](uint64_t t) { return sid[warp][t]; }, ld, lid, lane);
    }
    __syncthreads();
    md[warp * 32 + lane] = ld;
    mi[warp * 32 + lane] = lid;
    __syncthreads();
    if (warp == 0) {
        for (uint32_t w = 1; w < kWarps; ++w) {
            for (uint32_t i = 0; i < a.k; ++i) {
                const double dv = md[w * 32 + i];
                if (dv == kInf) break;
                warp_insert(dv, mi[w * 32 + i], ld, lid, a.k, lane);
            }
        }
        if (lane < a.k) {
            a.out_ids[q * a.k + lane] = lid;
            a.out_dists[q * a.k + lane] = a.squared ? ld : __dsqrt_rn(ld);
        }
    }
}

// ---------------------------- int8 screen with a prefix bound, wide rows (128 < d <= 1024)
// rerank_q8p_kernel's stage 1 unchanged (the first 48 dims in one 64-byte read, the query's prefix
// words in registers). Stage 2 — the rest of a queued row (up to 61 words) — is a warp-cooperative
// pass instead of a ring of whole rows: for each queued row, lane l loads words l and 32 + l of its
// rest, folds them against the query words it holds in registers, and a warp reduction gives the
// row's exact int8 dot product, four rows' loads in flight at a time. The full certified bounds,
// the shared tau and the exact fp64 survivors are rerank_q8p_kernel's. At cfg3 (d = 960) the first
// 48 dims rule out about 90 % of the candidates against the final tau (tools/partial_bound.py): a
// candidate costs 64 bytes instead of the 3,840 of its f32 row.
__global__ void __launch_bounds__(kThreads, 2) rerank_q8w_kernel(RerankArgs a, uint32_t stride) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr uint32_t kP = 3;               // prefix words
    constexpr uint32_t suA = kP + 2;         // meta0 + prefix words + 1: odd 16-byte stride
    double* qd = reinterpret_cast<double*>(smem);  // d
    const uint32_t ringA = kQ8Stages * 32 * suA;   // uint4 units
    const uint32_t per_warp = max(ringA * 16, kRows * stride * 4);
    unsigned char* wbase = smem + ((a.d * 8 + 15) / 16) * 16;
    __shared__ uint32_t qpack[256];          // the query's int8 words (d <= 1024)
    __shared__ uint32_t sid[kWarps][kQ8Cap];
    __shared__ float slo[kWarps][kQ8Cap];
    __shared__ uint32_t qqid[kWarps][kQ8QCap];
    __shared__ int qqI[kWarps][kQ8QCap];
    __shared__ double md[kWarps * 32];
    __shared__ uint32_t mi[kWarps * 32];
    __shared__ double qred[8][5];            // per warp: e2, b2, n2, e2s, b2s
    __shared__ double qpar[7];  // t, |q|^2, ||t b|| (up), ||e_q|| (up), t^2 |b_S|^2, ||e_q,S|| (up), t^2 |b|^2
    __shared__ double tau_cta;
    __shared__ unsigned long long tau_sh;
    __shared__ float qmax_sh[kWarps];
    __shared__ int ovf, qok;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    uint64_t q;
    if (!rerank_query(a, q)) return;
    const float* query = a.queries + q * a.d;
    const uint32_t nwq = a.qpad / 16, nr = nwq - kP;  // rest words
    for (uint32_t i = tid; i < a.d; i += kThreads) qd[i] = static_cast<double>(query[i]);
    // quantise the query: t = max|q| / 127 over the whole CTA; thread owns dims 4 tid .. 4 tid + 3
    float v[4], mx = 0.f;
#pragma unroll
    for (uint32_t j = 0; j < 4; ++j) {
        const uint32_t i = 4 * tid + j;
        v[j] = i < a.d ? query[i] : 0.f;
        mx = fmaxf(mx, fabsf(v[j]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, o));
    if (lane == 0) qmax_sh[warp] = mx;
    __syncthreads();
    mx = 0.f;
    for (uint32_t w = 0; w < kWarps; ++w) mx = fmaxf(mx, qmax_sh[w]);
    const float tq = mx / 127.f;
    {
        double e2 = 0.0, b2 = 0.0, n2 = 0.0;
        uint32_t packed = 0;
#pragma unroll
        for (uint32_t j = 0; j < 4; ++j) {
            const float bq = tq > 0.f ? fminf(127.f, fmaxf(-127.f, rintf(v[j] / tq))) : 0.f;
            const double e = static_cast<double>(v[j]) - static_cast<double>(tq) * static_cast<double>(bq);
            e2 += e * e;
            b2 += static_cast<double>(bq) * static_cast<double>(bq);
            n2 += static_cast<double>(v[j]) * static_cast<double>(v[j]);
            packed |= (static_cast<uint32_t>(static_cast<int>(bq)) & 0xffu) << (8 * j);
        }
        const bool pre = tid < 4 * kP;  // this thread's dims are in the prefix
        double e2s = pre ? e2 : 0.0, b2s = pre ? b2 : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            e2 += __shfl_xor_sync(kFull, e2, o);
            b2 += __shfl_xor_sync(kFull, b2, o);
            n2 += __shfl_xor_sync(kFull, n2, o);
            e2s += __shfl_xor_sync(kFull, e2s, o);
            b2s += __shfl_xor_sync(kFull, b2s, o);
        }
        qpack[tid] = packed;
        if (lane == 0) {
            qred[warp][0] = e2;
            qred[warp][1] = b2;
            qred[warp][2] = n2;
            qred[warp][3] = e2s;
            qred[warp][4] = b2s;
        }
    }
    __syncthreads();
    if (tid == 0) {
        double e2 = 0.0, b2 = 0.0, n2 = 0.0, e2s = 0.0, b2s = 0.0;
        for (uint32_t w = 0; w < kWarps; ++w) {
            e2 += qred[w][0];
            b2 += qred[w][1];
            n2 += qred[w][2];
            e2s += qred[w][3];
            b2s += qred[w][4];
        }
        qpar[0] = static_cast<double>(tq);
        qpar[1] = n2;
        qpar[2] = static_cast<double>(tq) * sqrt(b2) * (1.0 + 1e-12);
        qpar[3] = sqrt(e2) * (1.0 + 1e-12);
        qpar[4] = static_cast<double>(tq) * static_cast<double>(tq) * b2s;
        qpar[5] = sqrt(e2s) * (1.0 + 1e-12);
        qpar[6] = static_cast<double>(tq) * static_cast<double>(tq) * b2;
        qok = isfinite(n2) && isfinite(e2) && isfinite(qpar[2]);
        ovf = 0;
        tau_sh = 0x7ff0000000000000ull;
    }
    __syncthreads();
    int qv[kP][4];
#pragma unroll
    for (uint32_t w = 0; w < kP; ++w) {
#pragma unroll
        for (uint32_t j = 0; j < 4; ++j) qv[w][j] = static_cast<int>(qpack[4 * w + j]);
    }
    // this lane's query rest words: kP + lane and kP + 32 + lane
    int qr[2][4];
#pragma unroll
    for (uint32_t u = 0; u < 2; ++u) {
        const uint32_t w = kP + 32 * u + lane;
#pragma unroll
        for (uint32_t j = 0; j < 4; ++j) qr[u][j] = w < nwq ? static_cast<int>(qpack[4 * w + j]) : 0;
    }
    const double qt = qpar[0], rq = qpar[3], tb2S = qpar[4], eqS = qpar[5], tb2 = qpar[6];
    const bool qfin = qok != 0;
    uint4* ra = reinterpret_cast<uint4*>(wbase + warp * per_warp);
    uint32_t* qid = qqid[warp];
    int* qI = qqI[warp];
    const uint32_t* cands = a.cands + q * a.m;
    const uint64_t mq = a.counts ? a.counts[q] : a.m;
    const uint64_t first = uint64_t(warp) * 32;
    const uint64_t steps = mq > first ? (mq - first + 32 * kWarps - 1) / (32 * kWarps) : 0;
    auto sbase = [&](uint64_t g) { return first + g * 32 * kWarps; };
    auto load_id = [&](uint64_t g) -> uint32_t {
        const uint64_t i = sbase(g) + lane;
        if (g >= steps || i >= mq) return 0u;
        return a.identity ? static_cast<uint32_t>(i) : __ldcs(cands + i);
    };
    uint32_t id0 = load_id(0), id1 = load_id(1);
    auto issue_a = [&](uint64_t g) {  // the first 64 bytes of the step's 32 rows
        const uint32_t myid = (g & 1u) ? id1 : id0;
        uint4* st = ra + static_cast<uint32_t>(g % kQ8Stages) * 32 * suA;
        const uint64_t b = sbase(g);
#pragma unroll
        for (uint32_t t = lane; t < 32 * (kP + 1); t += 32) {
            const uint32_t row = t / (kP + 1), col = t % (kP + 1);
            const uint32_t id = __shfl_sync(kFull, myid, row);
            if (b + row < mq) cp_async16(st + row * suA + col, a.q8 + uint64_t(id) * a.qsplit + 16u * col);
        }
        if (g & 1u) id1 = load_id(g + 2);
        else id0 = load_id(g + 2);
        return myid;
    };
    uint32_t rowid0 = 0, rowid1 = 0;
    if (steps) rowid0 = issue_a(0);
    cp_async_commit();
    double sl = kInf;  // this warp's k smallest upper bounds (lane i = entry i)
    uint32_t nsurv = 0, qn = 0;
    bool overflow = false;
    auto tau_now = [&]() {
        const double own = __shfl_sync(kFull, sl, a.k - 1);
        const double shared = __longlong_as_double(static_cast<long long>(*reinterpret_cast<volatile unsigned long long*>(&tau_sh)));
        return fmin(own, shared);
    };
    // stage 2 over the queued rows [0, cnt): warp-cooperative rest-of-row dot products, 4 rows at a time
    auto drain = [&](uint32_t cnt) {
        for (uint32_t r0 = 0; r0 < cnt; r0 += 4) {
            uint4 x[4][2], mw[4];
            uint32_t rid[4];
            int rI[4];
#pragma unroll
            for (uint32_t u = 0; u < 4; ++u) {
                const bool live = r0 + u < cnt;
                rid[u] = live ? qid[r0 + u] : 0u;
                rI[u] = live ? qI[r0 + u] : 0;
                const int8_t* rec = a.q8b + uint64_t(rid[u]) * (a.qrec - a.qsplit);
                x[u][0] = live && lane < nr ? __ldcs(reinterpret_cast<const uint4*>(rec) + lane) : make_uint4(0, 0, 0, 0);
                x[u][1] = live && 32 + lane < nr ? __ldcs(reinterpret_cast<const uint4*>(rec) + 32 + lane) : make_uint4(0, 0, 0, 0);
                mw[u] = live ? __ldcs(reinterpret_cast<const uint4*>(rec) + nr) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (uint32_t u = 0; u < 4; ++u) {
                if (r0 + u >= cnt) break;
                int c = 0;
#pragma unroll
                for (uint32_t h = 0; h < 2; ++h) {
                    c = __dp4a(static_cast<int>(x[u][h].x), qr[h][0], c);
                    c = __dp4a(static_cast<int>(x[u][h].y), qr[h][1], c);
                    c = __dp4a(static_cast<int>(x[u][h].z), qr[h][2], c);
                    c = __dp4a(static_cast<int>(x[u][h].w), qr[h][3], c);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
                const int I = rI[u] + c;
                const float rR = __uint_as_float(mw[u].y), rs = __uint_as_float(mw[u].z);  // (|a|^2, ||e_x||, s, 0)
                double lo = 0.0, up = kInf;
                if (qfin && rs >= 0.f)
                    tri_bounds(static_cast<double>(rs), static_cast<double>(mw[u].x), tb2, qt, I, static_cast<double>(rR),
                               rq, lo, up);
                if (up < __shfl_sync(kFull, sl, a.k - 1)) {  // (uniform across the warp)
                    list_insert_val(up, sl, a.k, lane);
                    const double own = __shfl_sync(kFull, sl, a.k - 1);
                    if (lane == 0 && own < kInf && own >= 0.0)
                        atomicMin(&tau_sh, static_cast<unsigned long long>(__double_as_longlong(own)));
                }
                const double tau2 = tau_now();
                if (lo <= tau2 && !overflow) {
                    if (nsurv >= kQ8Cap) {  // drop buffered rows the tighter tau now excludes
                        const double tau = tau_now();
                        uint32_t kept = 0;
                        for (uint32_t t0 = 0; t0 < nsurv; t0 += 32) {
                            const uint32_t t = t0 + lane;
                            const bool in = t < nsurv;
                            const uint32_t idv = in ? sid[warp][t] : 0u;
                            const float lv = in ? slo[warp][t] : 0.f;
                            const bool keep = in && static_cast<double>(lv) <= tau;
                            const uint32_t kb = __ballot_sync(kFull, keep);
                            __syncwarp();
                            if (keep) {
                                const uint32_t p = kept + __popc(kb & ((1u << lane) - 1u));
                                sid[warp][p] = idv;
                                slo[warp][p] = lv;
                            }
                            kept += __popc(kb);
                            __syncwarp();
                        }
                        nsurv = kept;
                    }
                    if (nsurv >= kQ8Cap) {
                        overflow = true;
                    } else {
                        if (lane == 0) {
                            sid[warp][nsurv] = rid[u];
                            slo[warp][nsurv] = __double2float_rd(lo);
                        }
                        ++nsurv;
                    }
                    __syncwarp();
                }
            }
        }
    };
    PrefixGate gate;
    for (uint64_t g = 0; g < steps; ++g) {
        if (g + 1 < steps) {
            const uint32_t v2 = issue_a(g + 1);
            if (g & 1u) rowid0 = v2;
            else rowid1 = v2;
        }
        cp_async_commit();
        cp_async_wait<1>();  // the prefix step g has landed
        __syncwarp();
        // stage 1: the prefix bound of step g's rows
        const uint32_t myid = (g & 1u) ? rowid1 : rowid0;
        const uint4* row = ra + static_cast<uint32_t>(g % kQ8Stages) * 32 * suA + lane * suA;
        const uint4 m0 = row[0];
        int c0 = 0, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
        for (uint32_t w = 0; w < kP; ++w) {
            const uint4 x = row[1 + w];
            c0 = __dp4a(static_cast<int>(x.x), qv[w][0], c0);
            c1 = __dp4a(static_cast<int>(x.y), qv[w][1], c1);
            c2 = __dp4a(static_cast<int>(x.z), qv[w][2], c2);
            c3 = __dp4a(static_cast<int>(x.w), qv[w][3], c3);
        }
        __syncwarp();  // the slot is refilled by the next issue
        const int IS = (c0 + c1) + (c2 + c3);
        const float rs = __uint_as_float(m0.x), eS = __uint_as_float(m0.z);
        const bool valid = sbase(g) + lane < mq;
        gate.update(tau_now(), eqS);  // (every lane: the shuffle inside must not sit in an && chain)
        bool under = true;  // the prefix bound is within tau (PrefixGate: no square root per row)
        if (qfin && rs >= 0.f) {
            const double sv = static_cast<double>(rs);
            const double sa = sv * sv * static_cast<double>(m0.y);
            const double cr = 2.0 * sv * qt * static_cast<double>(IS);
            const double V = sa + tb2S - cr - 1.1368683772161603e-13 * (sa + tb2S + fabs(cr));
            under = gate.keeps(V, eS);
        }
        const uint32_t keep = __ballot_sync(kFull, valid && under);
        if (keep) {
            if ((keep >> lane) & 1u) {
                const uint32_t p = qn + __popc(keep & ((1u << lane) - 1u));
                qid[p] = myid;
                qI[p] = IS;
            }
            qn += __popc(keep);
            __syncwarp();
        }
        if (qn >= 32) {  // stage 2 of 32 queued rows (the rest moves to the front)
            drain(32);
            const uint32_t r0v = 32 + lane < qn ? qid[32 + lane] : 0u;
            const int r1v = 32 + lane < qn ? qI[32 + lane] : 0;
            __syncwarp();
            if (32 + lane < qn) {
                qid[lane] = r0v;
                qI[lane] = r1v;
            }
            __syncwarp();
            qn -= 32;
        }
    }
    if (qn) drain(qn);
    cp_async_wait<0>();
    if (overflow && lane == 0) atomicOr(&ovf, 1);
    md[warp * 32 + lane] = sl;
    __syncthreads();
    if (warp == 0) {
        for (uint32_t w = 1; w < kWarps; ++w) {
            for (uint32_t i = 0; i < a.k; ++i) {
                const double vv = md[w * 32 + i];
                if (!(vv < __shfl_sync(kFull, sl, a.k - 1))) break;  // lists are sorted
                list_insert_val(vv, sl, a.k, lane);
            }
        }
        const double t = __shfl_sync(kFull, sl, a.k - 1);
        if (lane == 0) tau_cta = t;
    }
    __syncthreads();
    const double tau = tau_cta;
    double ld = kInf;
    uint32_t lid = 0xffffffffu;
    float* st = reinterpret_cast<float*>(ra);  // the drained ring is staging now
    if (ovf) {  // exact re-rank of the whole query, the warps splitting the candidates
        const uint64_t per = (mq + kWarps - 1) / kWarps, lo = min_u64(mq, warp * per), hi = min_u64(mq, lo + per);
        if (a.screen_stats && tid == 0) atomicAdd(a.screen_stats + 1, 1ull);
        exact_rows(a, st, stride, qd, hi - lo,
                   [&](uint64_t t) { return a.identity ? static_cast<uint32_t>(lo + t) : cands[lo + t]; }, ld, lid, lane);
    } else {
        uint32_t kept = 0;
        for (uint32_t t0 = 0; t0 < nsurv; t0 += 32) {
            const uint32_t t = t0 + lane;
            const bool in = t < nsurv;
            const uint32_t idv = in ? sid[warp][t] : 0u;
            const bool keep = in && static_cast<double>(slo[warp][t]) <= tau;
            const uint32_t kb = __ballot_sync(kFull, keep);
            __syncwarp();
            if (keep) sid[warp][kept + __popc(kb & ((1u << lane) - 1u))] = idv;
            kept += __popc(kb);
            __syncwarp();
        }
        if (a.screen_stats && lane == 0) atomicAdd(a.screen_stats, static_cast<unsigned long long>(kept));
        exact_rows(a, st, stride, qd, kept, [&](uint64_t t) { return sid[warp][t]; }, ld, lid, lane);
    }
    __syncthreads();
    md[warp * 32 + lane] = ld;
    mi[warp * 32 + lane] = lid;
    __syncthreads();
    if (warp == 0) {
        for (uint32_t w = 1; w < kWarps; ++w) {
            for (uint32_t i = 0; i < a.k; ++i) {
                const double dv = md[w * 32 + i];
                if (dv == kInf) break;
                warp_insert(dv, mi[w * 32 + i], ld, lid, a.k, lane);
            }
        }
        if (lane < a.k) {
            a.out_ids[q * a.k + lane] = lid;
            a.out_dists[q * a.k + lane] = a.squared ? ld : __dsqrt_rn(ld);
        }
    }
}

// ---------------------------------------------------------------- u8 rows
// Data certified integer in [0, 255] at upload and a query of the same kind:
// every (x - q)^2 is an integer and every partial sum stays below 2^32, so
// the integer sum — in ANY order — is the exact value of the reference's fp64
// 4-accumulator sum. Rows are read as bytes (a quarter of the fp32 traffic):
// L = lanes per row (16 bytes each), R = 32 / L rows per warp load, U loads in
// flight per lane; |x - q| and the 4-byte dot product are one VABSDIFF4 and
// one IDP.4A per word; L lanes reduce a row with log2(L) shuffles.

__device__ __forceinline__ uint4 ld_nc_u4(const uint8_t* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

template <uint32_t L, bool GENERIC>
__global__ void __launch_bounds__(kThreads, 6) rerank_u8_kernel(RerankArgs a) {
    constexpr uint32_t R = 32 / L;
    constexpr uint32_t U = L >= 4 ? 4 : L;  // loads in flight per lane, with at most 32 rows per step
    constexpr uint32_t kStep = R * U;       // rows per warp step (<= 32: one candidate id per lane)
    static_assert(kStep <= 32, "one candidate id per lane");
    __shared__ double md[kWarps * 32];
    __shared__ uint32_t mi[kWarps * 32];
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    uint64_t q;
    if (!rerank_query(a, q)) return;
    const float* query = a.queries + q * a.d;
    bool ok = true;
    for (uint32_t i = tid; i < a.d; i += kThreads) ok &= is_u8(query[i]);
    if (!__syncthreads_and(ok)) return;  // the fp32/fp64 kernel owns this query
    const uint32_t c = lane % L, g = lane / L;
    const bool live = 16u * c < a.dpad;  // L is dpad/16 rounded up to a power of two
    uint32_t qw[4];
#pragma unroll
    for (uint32_t w = 0; w < 4; ++w) {
        uint32_t v = 0;
#pragma unroll
        for (uint32_t b = 0; b < 4; ++b) {
            const uint32_t i = 16u * c + 4u * w + b;
            if (i < a.d) v |= static_cast<uint32_t>(query[i]) << (8u * b);
        }
        qw[w] = v;
    }
    const uint32_t* cands = a.cands + q * a.m;
    const uint64_t mq = a.counts ? a.counts[q] : a.m;
    double ld = kInf;
    uint32_t lid = 0xffffffffu;
    for (uint64_t base = static_cast<uint64_t>(warp) * kStep; base < mq; base += kStep * kWarps) {
        const uint32_t my = (lane < kStep && base + lane < mq)
                                ? (a.identity ? static_cast<uint32_t>(base + lane) : __ldcs(cands + base + lane))
                                : 0u;
        uint32_t idr[U];
        bool vr[U];
        uint4 x[U];
#pragma unroll
        for (uint32_t u = 0; u < U; ++u) {
            const uint32_t r = u * R + g;
            idr[u] = __shfl_sync(kFull, my, r);
            vr[u] = base + r < mq;
            x[u] = (vr[u] && live) ? ld_nc_u4(a.data8 + static_cast<uint64_t>(idr[u]) * a.dpad + 16u * c)
                                   : make_uint4(0, 0, 0, 0);
        }
        double dist[U];
#pragma unroll
        for (uint32_t u = 0; u < U; ++u) {
            uint32_t acc = 0;
            acc = __dp4a(__vabsdiffu4(x[u].x, qw[0]), __vabsdiffu4(x[u].x, qw[0]), acc);
            acc = __dp4a(__vabsdiffu4(x[u].y, qw[1]), __vabsdiffu4(x[u].y, qw[1]), acc);
            acc = __dp4a(__vabsdiffu4(x[u].z, qw[2]), __vabsdiffu4(x[u].z, qw[2]), acc);
            acc = __dp4a(__vabsdiffu4(x[u].w, qw[3]), __vabsdiffu4(x[u].w, qw[3]), acc);
#pragma unroll
            for (uint32_t o = L / 2; o >= 1; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
            dist[u] = vr[u] ? static_cast<double>(acc) : kInf;
        }
        if constexpr (GENERIC) {
#pragma unroll
            for (uint32_t u = 0; u < U; ++u) {
                if (c == 0 && vr[u]) {
                    a.all_d[q * a.m + base + u * R + g] = dist[u];
                    a.all_id[q * a.m + base + u * R + g] = idr[u];
                }
            }
        } else {
#pragma unroll
            for (uint32_t u = 0; u < U; ++u) {
                const double wd = __shfl_sync(kFull, ld, a.k - 1);
                const uint32_t wi = __shfl_sync(kFull, lid, a.k - 1);
                uint32_t bal = __ballot_sync(kFull, c == 0 && vr[u] && dist_id_less(dist[u], idr[u], wd, wi));
                while (bal) {  // rows that beat the current k-th best (rare once the list fills)
                    const uint32_t src = __ffs(bal) - 1;
                    bal &= bal - 1;
                    warp_insert(__shfl_sync(kFull, dist[u], src), __shfl_sync(kFull, idr[u], src), ld, lid, a.k, lane);
                }
            }
        }
    }
    if constexpr (!GENERIC) {
        md[warp * 32 + lane] = ld;
        mi[warp * 32 + lane] = lid;
        __syncthreads();
        if (warp == 0) {
            for (uint32_t w = 1; w < kWarps; ++w) {
                for (uint32_t i = 0; i < a.k; ++i) {
                    const double dv = md[w * 32 + i];
                    if (dv == kInf) break;
                    warp_insert(dv, mi[w * 32 + i], ld, lid, a.k, lane);
                }
            }
            if (lane < a.k) {
                a.out_ids[q * a.k + lane] = lid;
                a.out_dists[q * a.k + lane] = a.squared ? ld : __dsqrt_rn(ld);
            }
        }
    }
}

// Pipelined byte rows (dpad <= 128): one candidate per lane. A warp step is 32 rows, copied
// global -> shared with coalesced 16-byte cp.async (8 lanes per 128-byte row) kU8Stages - 1 steps
// ahead, their ids loaded two steps before that; then every lane folds ITS row from shared memory
// (row stride an odd number of 16-byte units: conflict-free LDS.128) against the query words held in
// registers — VABSDIFF4 + IDP.4A per word, no cross-lane reduction — and one ballot per step finds
// the rows that beat the warp's k-th best.
constexpr uint32_t kU8Stages = 2;  // default ring depth (x 3 CTAs per SM); 3 x 2 via SUCO_U8_STAGES=3

template <uint32_t NW, bool GENERIC, uint32_t kU8Stages = kU8Stages, uint32_t MINB = 3>
__global__ void __launch_bounds__(kThreads, MINB) rerank_u8_pipe_kernel(RerankArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    uint64_t q;
    if (!rerank_query(a, q)) return;
    const float* query = a.queries + q * a.d;
    bool ok = true;
    for (uint32_t i = tid; i < a.d; i += kThreads) ok &= is_u8(query[i]);
    if (!__syncthreads_and(ok)) return;  // the fp32/fp64 kernel owns this query
    constexpr uint32_t nw = NW;                    // 16-byte units per row (dpad / 16 <= 8)
    constexpr uint32_t su = NW | 1u;               // row stride in 16-byte units (odd)
    __shared__ uint32_t qpack[32];                 // the query as bytes, packed once per CTA
    // (distance << 32 | id) of the best k-th entry over the CTA's warps: every warp already holds k
    // rows at or below its own k-th, so a row above this bound cannot reach the final top-k
    __shared__ unsigned long long kbound;
    if (tid == 0) kbound = ~0ull;
    if (tid < 32) {
        uint32_t v = 0;
#pragma unroll
        for (uint32_t b = 0; b < 4; ++b) {
            const uint32_t i = 4u * tid + b;
            if (i < a.d) v |= static_cast<uint32_t>(query[i]) << (8u * b);
        }
        qpack[tid] = v;
    }
    __syncthreads();
    uint4 qv[8];
#pragma unroll
    for (uint32_t w = 0; w < 8; ++w) qv[w] = reinterpret_cast<const uint4*>(qpack)[w];
    uint4* ring = reinterpret_cast<uint4*>(smem) + warp * kU8Stages * 32 * su;
    const uint32_t* cands = a.cands + q * a.m;
    const uint64_t mq = a.counts ? a.counts[q] : a.m;
    const uint64_t first = uint64_t(warp) * 32;
    const uint64_t steps = mq > first ? (mq - first + 32 * kWarps - 1) / (32 * kWarps) : 0;
    auto sbase = [&](uint64_t g) { return first + g * 32 * kWarps; };
    auto load_id = [&](uint64_t g) -> uint32_t {
        const uint64_t i = sbase(g) + lane;
        if (g >= steps || i >= mq) return 0u;
        return a.identity ? static_cast<uint32_t>(i) : __ldcs(cands + i);
    };
    uint32_t id0 = load_id(0), id1 = load_id(1);  // ids of the steps g with g % 2 == 0 / 1 next in line
    auto issue = [&](uint64_t g) {
        const uint32_t myid = (g & 1u) ? id1 : id0;
        uint4* st = ring + static_cast<uint32_t>(g % kU8Stages) * 32 * su;
        const uint64_t b = sbase(g);
#pragma unroll
        for (uint32_t t = lane; t < 32 * nw; t += 32) {
            const uint32_t row = t / nw, col = t % nw;  // constant divisor
            const uint32_t id = __shfl_sync(kFull, myid, row);
            if (b + row < mq) cp_async16(st + row * su + col, a.data8 + uint64_t(id) * a.dpad + 16u * col);
        }
        if (g & 1u) id1 = load_id(g + 2);
        else id0 = load_id(g + 2);
        return myid;
    };
    uint32_t rowid[kU8Stages];  // each lane's row id per ring slot
#pragma unroll
    for (uint32_t i = 0; i < kU8Stages; ++i) rowid[i] = 0;
    for (uint32_t i = 0; i + 1 < kU8Stages; ++i) {
        if (i < steps) rowid[i] = issue(i);
        cp_async_commit();
    }
    double ld = kInf;
    uint32_t lid = 0xffffffffu;
    for (uint64_t g = 0; g < steps; ++g) {
        if (g + kU8Stages - 1 < steps) {
            const uint32_t v = issue(g + kU8Stages - 1);
            const uint32_t sl = static_cast<uint32_t>((g + kU8Stages - 1) % kU8Stages);
#pragma unroll
            for (uint32_t i = 0; i < kU8Stages; ++i) {
                if (i == sl) rowid[i] = v;
            }
        }
        cp_async_commit();
        cp_async_wait<kU8Stages - 1>();
        __syncwarp();
        const uint32_t sl = static_cast<uint32_t>(g % kU8Stages);
        uint32_t myid = rowid[0];
#pragma unroll
        for (uint32_t i = 1; i < kU8Stages; ++i) {
            if (i == sl) myid = rowid[i];
        }
        const uint4* row = ring + sl * 32 * su + lane * su;
        uint32_t c0 = 0, c1 = 0, c2 = 0, c3 = 0;  // four independent chains (integer sums: any order)
#pragma unroll
        for (uint32_t w = 0; w < nw; ++w) {
            const uint4 x = row[w];
            uint32_t t;
            t = __vabsdiffu4(x.x, qv[w].x);
            c0 = __dp4a(t, t, c0);
            t = __vabsdiffu4(x.y, qv[w].y);
            c1 = __dp4a(t, t, c1);
            t = __vabsdiffu4(x.z, qv[w].z);
            c2 = __dp4a(t, t, c2);
            t = __vabsdiffu4(x.w, qv[w].w);
            c3 = __dp4a(t, t, c3);
        }
        const uint32_t acc = (c0 + c1) + (c2 + c3);
        __syncwarp();  // the slot is refilled by the next step's issue
        const uint64_t b = sbase(g);
        const bool valid = b + lane < mq;
        const double dist = valid ? static_cast<double>(acc) : kInf;
        if constexpr (GENERIC) {
            if (valid) {
                a.all_d[q * a.m + b + lane] = dist;
                a.all_id[q * a.m + b + lane] = myid;
            }
        } else {
            const unsigned long long kb = *reinterpret_cast<volatile unsigned long long*>(&kbound);
            const unsigned long long key = (static_cast<unsigned long long>(acc) << 32) | myid;
            uint32_t bal = __ballot_sync(kFull, valid && key < kb);
            if (bal) {
                while (bal) {  // rows that beat the bound (rare once the lists fill)
                    const uint32_t src = __ffs(bal) - 1;
                    bal &= bal - 1;
                    warp_insert(__shfl_sync(kFull, dist, src), __shfl_sync(kFull, myid, src), ld, lid, a.k, lane);
                }
                const double wd = __shfl_sync(kFull, ld, a.k - 1);
                const uint32_t wi = __shfl_sync(kFull, lid, a.k - 1);
                if (lane == 0 && wd != kInf)  // integer distances below 2^32: exact as u32
                    atomicMin(&kbound, (static_cast<unsigned long long>(static_cast<uint32_t>(wd)) << 32) | wi);
            }
        }
    }
    cp_async_wait<0>();
    if constexpr (!GENERIC) {
        __syncthreads();  // every warp's copies are done: the ring becomes the merge area
        double* md = reinterpret_cast<double*>(smem);
        uint32_t* mi = reinterpret_cast<uint32_t*>(md + kWarps * 32);
        md[warp * 32 + lane] = ld;
        mi[warp * 32 + lane] = lid;
        __syncthreads();
        if (warp == 0) {
            for (uint32_t w = 1; w < kWarps; ++w) {
                for (uint32_t i = 0; i < a.k; ++i) {
                    const double dv = md[w * 32 + i];
                    if (dv == kInf) break;
                    warp_insert(dv, mi[w * 32 + i], ld, lid, a.k, lane);
                }
            }
            if (lane < a.k) {
                a.out_ids[q * a.k + lane] = lid;
                a.out_dists[q * a.k + lane] = a.squared ? ld : __dsqrt_rn(ld);
            }
        }
    }
}

// k > 32: k rounds of "smallest (dist, id) strictly after the previous pick"
// over the m scored candidates of one query; (dist, id) is a strict total
// order so this reproduces nth_element + sort (query.cpp:185-189).
__global__ void __launch_bounds__(256) topk_generic_kernel(RerankArgs a) {
    __shared__ double sd[8];
    __shared__ uint32_t si[8];
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    uint64_t q;
    if (!rerank_query(a, q)) return;
    const double* dd = a.all_d + q * a.m;
    const uint32_t* ii = a.all_id + q * a.m;
    const uint64_t mq = a.counts ? a.counts[q] : a.m;
    double pd = -1.0;
    uint32_t pi = 0;
    for (uint32_t r = 0; r < a.k; ++r) {
        double bd = kInf;
        uint32_t bi = 0xffffffffu;
        for (uint64_t c = tid; c < mq; c += 256) {
            const double d = dd[c];
            const uint32_t i = ii[c];
            if (dist_id_less(pd, pi, d, i) && dist_id_less(d, i, bd, bi)) {
                bd = d;
                bi = i;
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double od = __shfl_xor_sync(kFull, bd, off);
            const uint32_t oi = __shfl_xor_sync(kFull, bi, off);
            if (dist_id_less(od, oi, bd, bi)) {
                bd = od;
                bi = oi;
            }
        }
        if (lane == 0) {
            sd[warp] = bd;
            si[warp] = bi;
        }
        __syncthreads();
        bd = sd[0];
        bi = si[0];
        for (int w = 1; w < 8; ++w) {
            if (dist_id_less(sd[w], si[w], bd, bi)) {
                bd = sd[w];
                bi = si[w];
            }
        }
        __syncthreads();
        if (tid == 0) {
            a.out_ids[q * a.k + r] = bi;
            a.out_dists[q * a.k + r] = a.squared ? bd : __dsqrt_rn(bd);
        }
        pd = bd;
        pi = bi;
    }
}

// k > 32: the k smallest (dist, id) of a query's m scored candidates by MSB radix select on the
// distance bits (non-negative doubles order like their bit patterns): 8-bit digits narrow the
// bucket holding the k-th distance until it has at most kRxCap members (usually 3 passes over the
// m distances), then one pass gathers the bucket and every smaller distance into shared memory,
// where a bitonic sort by (dist, id) — a strict total order, so this is the reference's
// nth_element + sort (query.cpp:185-189) — yields the k. A bucket that never fits (masses of
// equal distances) or k > kRxCap / 2 takes the k-round kernel above.
constexpr uint32_t kRxCap = 2048;

__device__ __forceinline__ unsigned long long dbits(double d) {
    return static_cast<unsigned long long>(__double_as_longlong(d));
}

__global__ void __launch_bounds__(1024) topk_radix_kernel(RerankArgs a, uint32_t* fallback) {
    __shared__ uint32_t hist[256];
    __shared__ unsigned long long key[kRxCap];
    __shared__ uint32_t kid[kRxCap];
    __shared__ uint32_t nsel, sbin, sbefore;
    const uint32_t tid = threadIdx.x, nt = blockDim.x;
    uint64_t q;
    if (!rerank_query(a, q)) return;
    const double* dd = a.all_d + q * a.m;
    const uint32_t* ii = a.all_id + q * a.m;
    const uint64_t mq = a.counts ? a.counts[q] : a.m;
    const uint32_t kk = static_cast<uint32_t>(min_u64(a.k, mq));
    unsigned long long prefix = 0, mask = 0;
    uint32_t need = kk;           // rank of the k-th inside the current bucket (1-based)
    uint64_t lt = 0;              // elements below the bucket
    for (int shift = 56; shift >= 0 && kk; shift -= 8) {
        for (uint32_t b = tid; b < 256; b += nt) hist[b] = 0;
        __syncthreads();
        for (uint64_t c = tid; c < mq; c += nt) {
            const unsigned long long u = dbits(dd[c]);
            if ((u & mask) == prefix) atomicAdd(&hist[(u >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (tid < 32) {  // the bin holding rank `need`: warp scan over 8 bins per lane
            uint32_t loc[8], sum = 0;
#pragma unroll
            for (uint32_t j = 0; j < 8; ++j) {
                loc[j] = hist[tid * 8 + j];
                sum += loc[j];
            }
            uint32_t incl = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(kFull, incl, o);
                if (tid >= static_cast<uint32_t>(o)) incl += y;
            }
            uint32_t run = incl - sum;
#pragma unroll
            for (uint32_t j = 0; j < 8; ++j) {
                if (run < need && need <= run + loc[j]) {
                    sbin = tid * 8 + j;
                    sbefore = run;
                }
                run += loc[j];
            }
        }
        __syncthreads();
        const uint32_t bin = sbin, before = sbefore;
        need -= before;
        lt += before;
        prefix |= static_cast<unsigned long long>(bin) << shift;
        mask |= 255ull << shift;
        if (hist[bin] + lt <= kRxCap) break;  // bucket + everything below it fits shared memory
        __syncthreads();
    }
    // gather: every element below the bucket, and the bucket
    if (tid == 0) nsel = 0;
    __syncthreads();
    const bool fits = kk == 0 || lt + hist[sbin] <= kRxCap;
    if (fits) {
        for (uint64_t c = tid; c < mq; c += nt) {
            const unsigned long long u = dbits(dd[c]);
            if ((u & mask) < prefix || (u & mask) == prefix) {
                // below the bucket: a prefix-masked value below the bucket's prefix means u is smaller
                const uint32_t pos = atomicAdd(&nsel, 1u);
                if (pos < kRxCap) {
                    key[pos] = u;
                    kid[pos] = ii[c];
                }
            }
        }
    }
    __syncthreads();
    if (!fits || nsel > kRxCap) {  // a huge bucket of equal distances: the k-round kernel
        if (tid == 0) fallback[atomicAdd(fallback, 1u) + 1] = static_cast<uint32_t>(q);
        return;
    }
    // bitonic sort of nsel (<= kRxCap) entries by (dist bits, id), padded to a power of two
    const uint32_t n = nsel;
    uint32_t np2 = 1;
    while (np2 < n) np2 <<= 1;
    for (uint32_t i = n + tid; i < np2; i += nt) {
        key[i] = ~0ull;
        kid[i] = 0xffffffffu;
    }
    __syncthreads();
    for (uint32_t size = 2; size <= np2; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = tid; i < np2; i += nt) {
                const uint32_t j = i ^ stride;
                if (j > i) {
                    const bool up = (i & size) == 0;
                    const bool gt = key[i] > key[j] || (key[i] == key[j] && kid[i] > kid[j]);
                    if (gt == up) {
                        const unsigned long long tk = key[i];
                        key[i] = key[j];
                        key[j] = tk;
                        const uint32_t ti = kid[i];
                        kid[i] = kid[j];
                        kid[j] = ti;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (uint32_t r = tid; r < a.k; r += nt) {
        const bool in = r < kk;
        const double dv = in ? __longlong_as_double(static_cast<long long>(key[r])) : kInf;
        a.out_ids[q * a.k + r] = in ? kid[r] : 0xffffffffu;
        a.out_dists[q * a.k + r] = a.squared || !in ? dv : __dsqrt_rn(dv);
    }
}

}  // namespace

// k > 32 selection over the scored candidates: radix select, the k-round kernel for the rest
static cudaError_t launch_topk(const RerankArgs& a, uint64_t nq, cudaStream_t st) {
    if (a.k > kRxCap / 2 || a.qlist) {
        topk_generic_kernel<<<static_cast<unsigned>(nq), 256, 0, st>>>(a);
        return cudaGetLastError();
    }
    uint32_t* fb = nullptr;  // [count, queries...] of the queries the radix kernel hands back
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&fb), (nq + 1) * 4, st);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(fb, 0, 4, st);
    if (e == cudaSuccess) {
        topk_radix_kernel<<<static_cast<unsigned>(nq), 1024, 0, st>>>(a, fb);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) {
        RerankArgs b = a;
        b.qlist = fb + 1;
        b.nlist = fb;
        b.qskip = nullptr;
        topk_generic_kernel<<<static_cast<unsigned>(nq), 256, 0, st>>>(b);  // CTAs past *nlist exit at once
        e = cudaGetLastError();
    }
    cudaFreeAsync(fb, st);
    return e;
}

cudaError_t launch_rerank(const RerankArgs& a, uint64_t nq, cudaStream_t st) {
    if (nq == 0) return cudaSuccess;
    const size_t smem = ((a.d * 8 + 15) / 16) * 16 + ((a.d + 3) / 4) * 16 + static_cast<size_t>(kWarps) * kRows * kStride * 4;
    const bool vec = (a.d % 4) == 0;
    const bool generic = a.k > 32;
    auto launch = [&](auto kern) -> cudaError_t {
        if (smem > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
            if (e != cudaSuccess) return e;
        }
        kern<<<static_cast<unsigned>(nq), kThreads, smem, st>>>(a);
        return cudaGetLastError();
    };
    cudaError_t e = cudaSuccess;
    if (a.data8 && a.dpad <= 128 && !a.u8_regs) {
        const uint32_t nwr = a.dpad / 16, su = nwr | 1u;
        const size_t usmem = size_t(kWarps) * kU8Stages * 32 * su * 16;
        using K = void (*)(RerankArgs);
        const K kg[8] = {rerank_u8_pipe_kernel<1, true>, rerank_u8_pipe_kernel<2, true>, rerank_u8_pipe_kernel<3, true>,
                         rerank_u8_pipe_kernel<4, true>, rerank_u8_pipe_kernel<5, true>, rerank_u8_pipe_kernel<6, true>,
                         rerank_u8_pipe_kernel<7, true>, rerank_u8_pipe_kernel<8, true>};
        const K kn[8] = {rerank_u8_pipe_kernel<1, false>, rerank_u8_pipe_kernel<2, false>, rerank_u8_pipe_kernel<3, false>,
                         rerank_u8_pipe_kernel<4, false>, rerank_u8_pipe_kernel<5, false>, rerank_u8_pipe_kernel<6, false>,
                         rerank_u8_pipe_kernel<7, false>, rerank_u8_pipe_kernel<8, false>};
        K kern = generic ? kg[nwr - 1] : kn[nwr - 1];
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(usmem));
        if (e != cudaSuccess) return e;
        kern<<<static_cast<unsigned>(nq), kThreads, usmem, st>>>(a);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    } else if (a.data8) {  // u8 queries here; the fp32/fp64 kernel below takes the others
        uint32_t L = 1;
        while (L < a.dpad / 16) L <<= 1;
        auto u8 = [&](auto kg, auto kn) {
            (generic ? kg : kn)<<<static_cast<unsigned>(nq), kThreads, 0, st>>>(a);
            return cudaGetLastError();
        };
        switch (L) {
            case 1: e = u8(rerank_u8_kernel<1, true>, rerank_u8_kernel<1, false>); break;
            case 2: e = u8(rerank_u8_kernel<2, true>, rerank_u8_kernel<2, false>); break;
            case 4: e = u8(rerank_u8_kernel<4, true>, rerank_u8_kernel<4, false>); break;
            case 8: e = u8(rerank_u8_kernel<8, true>, rerank_u8_kernel<8, false>); break;
            case 16: e = u8(rerank_u8_kernel<16, true>, rerank_u8_kernel<16, false>); break;
            default: e = u8(rerank_u8_kernel<32, true>, rerank_u8_kernel<32, false>); break;
        }
        if (e != cudaSuccess) return e;
    }
    const int pmode = a.pipe == 0 ? 2 : a.pipe == 1 ? 1 : 0;  // 2 screened, 1 pipelined fp64, 0 unpipelined
    // int8 screen for long candidate lists only: with a few hundred candidates per query the fp32
    // screen is cheap and the int8 bounds prune little (measured, cfg1 m = 500: every candidate
    // survived the prefix bound, re-rank 0.27 ms vs 0.095 ms for the fp32 screen; cfg4 m = 50,000:
    // 7.9 ms vs 28.3 ms)
    if (vec && !generic && pmode == 2 && a.q8 && a.qpre == 3 && a.qpad > 128 && a.qpad <= 1024 &&
        a.m >= a.q8_min) {  // wide rows: the prefix screen with a warp-cooperative second stage
        const uint32_t stride = 32 * ((min(a.d, kChunk) + 31) / 32) + 4;
        const size_t rings = size_t(kQ8Stages) * 32 * 5 * 16;
        const size_t wsmem = ((a.d * 8 + 15) / 16) * 16 + kWarps * std::max<size_t>(rings, size_t(kRows) * stride * 4);
        e = cudaFuncSetAttribute(rerank_q8w_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(wsmem));
        if (e != cudaSuccess) return e;
        rerank_q8w_kernel<<<static_cast<unsigned>(nq), kThreads, wsmem, st>>>(a, stride);
        return cudaGetLastError();
    }
    if (vec && !generic && pmode == 2 && a.q8 && a.qpad >= 16 && a.qpad <= 128 && a.m >= a.q8_min) {
        const uint32_t stride = 32 * ((min(a.d, kChunk) + 31) / 32) + 4;
        const uint32_t nwq = a.qpad / 16, su = (nwq + 1) | 1u;
        const size_t per_warp = std::max<size_t>(size_t(kQ8Stages) * 32 * su * 16, size_t(kRows) * stride * 4);
        const size_t qsmem = ((a.d * 8 + 15) / 16) * 16 + kWarps * per_warp;
        using KQ = void (*)(RerankArgs, uint32_t);
        const KQ kt[8] = {rerank_q8_kernel<1, true>, rerank_q8_kernel<2, true>, rerank_q8_kernel<3, true>,
                          rerank_q8_kernel<4, true>, rerank_q8_kernel<5, true>, rerank_q8_kernel<6, true>,
                          rerank_q8_kernel<7, true>, rerank_q8_kernel<8, true>};
        const KQ kc[8] = {rerank_q8_kernel<1, false>, rerank_q8_kernel<2, false>, rerank_q8_kernel<3, false>,
                          rerank_q8_kernel<4, false>, rerank_q8_kernel<5, false>, rerank_q8_kernel<6, false>,
                          rerank_q8_kernel<7, false>, rerank_q8_kernel<8, false>};
        KQ kern = a.no_tma ? kc[nwq - 1] : kt[nwq - 1];
        size_t ksmem = qsmem;
        if (a.qpre) {  // the prefix-bound kernel (records in its layout, pack_q8_kernel)
            const KQ k1[7] = {rerank_q8p_kernel<1, 1>, rerank_q8p_kernel<1, 2>, rerank_q8p_kernel<1, 3>,
                              rerank_q8p_kernel<1, 4>, rerank_q8p_kernel<1, 5>, rerank_q8p_kernel<1, 6>,
                              rerank_q8p_kernel<1, 7>};
            const KQ k3[5] = {rerank_q8p_kernel<3, 1>, rerank_q8p_kernel<3, 2>, rerank_q8p_kernel<3, 3>,
                              rerank_q8p_kernel<3, 4>, rerank_q8p_kernel<3, 5>};
            kern = a.qpre == 1 ? k1[nwq - 2] : k3[nwq - 4];
            const uint32_t nr = nwq - a.qpre, sub = (nr + 1) | 1u, sua = (a.qpre + 1) | 1u;
            const size_t rings = (size_t(kQ8Stages) * 32 * sua + size_t(2) * 32 * sub) * 16;
            ksmem = ((a.d * 8 + 15) / 16) * 16 + kWarps * std::max<size_t>(rings, size_t(kRows) * stride * 4);
        }
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(ksmem));
        if (e != cudaSuccess) return e;
        kern<<<static_cast<unsigned>(nq), kThreads, ksmem, st>>>(a, stride);
        return cudaGetLastError();
    }
    if (vec && !generic && pmode == 2) {
        const uint32_t stride = 32 * ((min(a.d, kChunk) + 31) / 32) + 4;  // = 4 (mod 32): conflict-free chains
        const size_t qbytes = ((a.d * 4 + 15) / 16) * 16 + ((a.d * 8 + 15) / 16) * 16;
        const size_t s3 = qbytes + size_t(kWarps) * 3 * kRows * stride * 4;
        const size_t s2 = qbytes + size_t(kWarps) * 2 * kRows * stride * 4;
        // occupancy first (measured: 2 stages x 3 CTAs per SM beat 3 x 2 for the byte rows): 3 CTAs
        // when 2 stages fit 60 KB (228 KB per SM, about 14 KB static + 1 KB reserved each), else 3
        // stages x 2 CTAs when that fits 98 KB, else 2 x 2.
        void (*kern)(RerankArgs, uint32_t) = rerank_screen_kernel<2, 2>;
        size_t ssmem = s2;
        if (s2 <= 60 * 1024) {
            kern = rerank_screen_kernel<2, 3>;
        } else if (s3 <= 98 * 1024) {
            kern = rerank_screen_kernel<3, 2>;
            ssmem = s3;
        }
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(ssmem));
        if (e != cudaSuccess) return e;
        kern<<<static_cast<unsigned>(nq), kThreads, ssmem, st>>>(a, stride);
        return cudaGetLastError();
    }
    if (vec && pmode != 0) {
        const size_t psmem = ((a.d * 8 + 15) / 16) * 16 + ((a.d + 3) / 4) * 16 +
                             static_cast<size_t>(kWarps) * kStages * kRows * kStride * 4;
        auto kern = generic ? rerank_pipe_kernel<true> : rerank_pipe_kernel<false>;
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(psmem));
        if (e != cudaSuccess) return e;
        kern<<<static_cast<unsigned>(nq), kThreads, psmem, st>>>(a);
        e = cudaGetLastError();
    } else if (vec) {
        e = generic ? launch(rerank_kernel<true, true>) : launch(rerank_kernel<true, false>);
    } else {
        e = generic ? launch(rerank_kernel<false, true>) : launch(rerank_kernel<false, false>);
    }
    if (e != cudaSuccess || !generic) return e;
    return launch_topk(a, nq, st);
}

}  // namespace suco_gpu
