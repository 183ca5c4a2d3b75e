// Shard-local kernels of the multi-GPU query protocol.
//
// Points are partitioned block-cyclically: with block size b and G shards,
// global block j = ids [j*b, (j+1)*b) lives on shard j % G. A shard keeps its
// blocks back to back in a local id space (local l <-> global
// ((l / b) * G + shard) * b + l % b), and keeps the GLOBAL per-cell sizes so
// that every shard's Dynamic Activation cut is the global one.
//
// Phase 1 (per query): local SC-scores (u8, one byte per local point) and,
// per local block, #points with score >= t for t = 0..N_s+1 (t = 0 is the
// block length). After the cross-shard exchange (host / NCCL), phase 2 takes
// the global threshold T and, per local block, the tie quota in global id
// order, and emits the local candidates: every score > T plus the first
// quota ties (score == T) of the block in id order — i.e. exactly the
// reference's top-m by (score desc, id asc) restricted to this shard.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.h"

namespace suco_gpu {
namespace {

constexpr uint32_t kFull = 0xffffffffu;

// hist[q][blk][t] = #local points of block blk with score >= t (t <= ns + 1).
// 16 scores per thread-step (uint4), SWAR high-bit tests per level (scores <= 127).
__global__ void __launch_bounds__(256) block_hist_kernel(const uint8_t* __restrict__ scores, uint64_t n_local,
                                                         uint64_t sstride, uint32_t b, uint32_t nblocks, uint32_t ns,
                                                         uint32_t* __restrict__ hist) {
    extern __shared__ uint32_t hs[];  // ns + 2
    const uint64_t q = blockIdx.y;
    const uint32_t blk = blockIdx.x;
    for (uint32_t t = threadIdx.x; t < ns + 2; t += blockDim.x) hs[t] = 0;
    __syncthreads();
    const uint64_t lo = uint64_t(blk) * b;
    const uint32_t len = static_cast<uint32_t>(min_u64(b, n_local - lo));
    const uint8_t* sc = scores + q * sstride + lo;
    const bool vec = ((reinterpret_cast<uintptr_t>(sc) & 15u) == 0) && ns <= 127;
    if (vec) {
        const uint32_t nv = len / 16;
        for (uint32_t t = 1; t <= ns; ++t) {
            const uint32_t kq = (0x80u - t) * 0x01010101u;
            uint32_t c = 0;
            for (uint32_t i = threadIdx.x; i < nv; i += blockDim.x) {
                const uint4 v = reinterpret_cast<const uint4*>(sc)[i];
                c += __popc((v.x + kq) & 0x80808080u) + __popc((v.y + kq) & 0x80808080u) +
                     __popc((v.z + kq) & 0x80808080u) + __popc((v.w + kq) & 0x80808080u);
            }
            for (uint32_t i = nv * 16 + threadIdx.x; i < len; i += blockDim.x) c += sc[i] >= t;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
            if ((threadIdx.x & 31) == 0 && c) atomicAdd(hs + t, c);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t* out = hist + (q * nblocks + blk) * (ns + 2);
            out[0] = len;
            for (uint32_t t = 1; t <= ns; ++t) out[t] = hs[t];
            out[ns + 1] = 0;
        }
        return;
    }
    for (uint32_t i = threadIdx.x; i < len; i += blockDim.x) {
        const uint32_t v = sc[i];
        if (v) atomicAdd(hs + v, 1u);  // exact-value counts, suffix-summed below
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t* out = hist + (q * nblocks + blk) * (ns + 2);
        uint32_t run = 0;
        out[ns + 1] = 0;
        for (uint32_t t = ns; t >= 1; --t) {
            run += hs[t];
            out[t] = run;
        }
        out[0] = len;
    }
}

// Vector forms (16-byte aligned score rows and blocks): one WARP per (query,
// block), lanes read consecutive uint4s (512 coalesced bytes per warp step).
__device__ __forceinline__ uint32_t ge_count16(const uint4 v, uint32_t t) {  // #bytes >= t, bytes <= 127
    const uint32_t kq = (0x80u - t) * 0x01010101u;
    return __popc((v.x + kq) & 0x80808080u) + __popc((v.y + kq) & 0x80808080u) + __popc((v.z + kq) & 0x80808080u) +
           __popc((v.w + kq) & 0x80808080u);
}

template <uint32_t NSB>
__global__ void __launch_bounds__(256) block_hist_vec_kernel(const uint8_t* __restrict__ scores, uint64_t n_local,
                                                             uint64_t sstride, uint32_t b, uint32_t nblocks,
                                                             uint32_t ns, uint32_t* __restrict__ hist) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t blk = blockIdx.x * 8 + (threadIdx.x >> 5);
    const uint64_t q = blockIdx.y;
    if (blk >= nblocks) return;
    const uint64_t lo = uint64_t(blk) * b;
    const uint32_t len = static_cast<uint32_t>(min_u64(b, n_local - lo));
    const uint4* sc = reinterpret_cast<const uint4*>(scores + q * sstride + lo);
    const uint32_t nv = len / 16;  // len % 16 != 0 only for the shard's last block
    uint32_t c[NSB];
#pragma unroll
    for (uint32_t t = 0; t < NSB; ++t) c[t] = 0;
    for (uint32_t i = lane; i < nv; i += 32) {
        const uint4 v = __ldcs(sc + i);
#pragma unroll
        for (uint32_t t = 0; t < NSB; ++t) c[t] += ge_count16(v, t + 1);
    }
    for (uint32_t i = nv * 16 + lane; i < len; i += 32) {
        const uint32_t v = reinterpret_cast<const uint8_t*>(sc)[i];
#pragma unroll
        for (uint32_t t = 0; t < NSB; ++t) c[t] += v >= t + 1;
    }
#pragma unroll
    for (uint32_t t = 0; t < NSB; ++t) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c[t] += __shfl_xor_sync(kFull, c[t], o);
    }
    uint32_t* out = hist + (q * nblocks + blk) * (ns + 2);
#pragma unroll
    for (uint32_t t = 0; t < NSB; ++t) {
        if (lane == t && t < ns) out[t + 1] = c[t];
    }
    if (lane == 0) {
        out[0] = len;
        out[ns + 1] = 0;
    }
}

__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t x, uint32_t lane, uint32_t& total) {
    uint32_t y = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t z = __shfl_up_sync(kFull, y, o);
        if (lane >= (uint32_t)o) y += z;
    }
    total = __shfl_sync(kFull, y, 31);
    return y - x;
}

// Warp per (query, block): every score > T plus the first `quota` ties in id
// order; lanes own consecutive 16-byte groups, so (warp step, lane, byte) is id order.
__global__ void __launch_bounds__(256) shard_emit_vec_kernel(const uint8_t* __restrict__ scores, uint64_t n_local,
                                                             uint64_t sstride, uint32_t b, uint32_t nblocks,
                                                             uint32_t shard, uint32_t num_shards,
                                                             const uint32_t* __restrict__ T,
                                                             const uint32_t* __restrict__ quota,
                                                             const uint32_t* __restrict__ base,
                                                             uint32_t* __restrict__ cands, uint64_t stride) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t blk = blockIdx.x * 8 + (threadIdx.x >> 5);
    const uint64_t q = blockIdx.y;
    if (blk >= nblocks) return;
    const uint64_t lo = uint64_t(blk) * b;
    const uint32_t len = static_cast<uint32_t>(min_u64(b, n_local - lo));
    const uint8_t* sc = scores + q * sstride + lo;
    const uint32_t t = T[q];
    const uint32_t qu = quota[q * nblocks + blk];
    uint32_t* out = cands + q * stride + base[q * nblocks + blk];
    const uint32_t gbase = static_cast<uint32_t>(lo);  // local ids (rerank reports global ids)
    const uint32_t ngroups = (len + 15) / 16;
    const uint32_t nfull = len / 16;
    uint32_t taken_run = 0, tie_run = 0;  // warp-uniform running totals
    constexpr uint32_t kU = 4;            // 16-byte loads in flight per lane
    for (uint32_t g0 = 0; g0 < ngroups; g0 += 32 * kU) {
        uint4 vv[kU];
#pragma unroll
        for (uint32_t u = 0; u < kU; ++u) {
            const uint32_t gi = g0 + u * 32 + lane;
            vv[u] = gi < nfull ? __ldcs(reinterpret_cast<const uint4*>(sc) + gi) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (uint32_t u = 0; u < kU; ++u) {
            const uint32_t gi = g0 + u * 32 + lane;
            if (g0 + u * 32 >= ngroups) break;  // warp-uniform
            const uint32_t valid = gi < ngroups ? min(16u, len - gi * 16) : 0u;
            uint4 v = vv[u];
            uint32_t ge = 0, gt = 0;
            if (valid == 16) {
                ge = ge_count16(v, t);
                gt = ge_count16(v, t + 1);
            } else if (valid) {  // ragged tail of the shard's last block: count valid bytes only (T may be 0)
                uint8_t tmp[16];
#pragma unroll
                for (uint32_t j = 0; j < 16; ++j) {
                    tmp[j] = j < valid ? sc[gi * 16 + j] : 0;
                    ge += j < valid && tmp[j] >= t;
                    gt += j < valid && tmp[j] > t;
                }
                v = *reinterpret_cast<uint4*>(tmp);
            }
            const uint32_t nt = ge - gt;  // ties
            if (!__any_sync(kFull, gt | (nt && tie_run < qu))) {
                tie_run += __reduce_add_sync(kFull, nt);
                continue;
            }
            uint32_t ties_total;
            const uint32_t tie_before = tie_run + warp_excl_scan(nt, lane, ties_total);
            const uint32_t tie_take = tie_before >= qu ? 0u : min(nt, qu - tie_before);
            uint32_t taken_total;
            const uint32_t pos0 = taken_run + warp_excl_scan(gt + tie_take, lane, taken_total);
            if (gt + tie_take) {
                uint32_t pos = pos0, tk = tie_take;
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (uint32_t j = 0; j < 16; ++j) {
                    const uint32_t s = (w[j >> 2] >> (8 * (j & 3))) & 0xffu;
                    if (j < valid && (s > t || (s == t && tk))) {
                        if (s == t) --tk;
                        out[pos++] = gbase + gi * 16 + j;
                    }
                }
            }
            tie_run += ties_total;
            taken_run += taken_total;
        }
    }
}

// One CTA per (query, local block): every score > T and the first `quota`
// ties (score == T) of the block, in id order, as GLOBAL ids at
// cands[q][base[q][blk] ...). Each thread owns a contiguous run of scores.
__global__ void __launch_bounds__(256) shard_emit_kernel(const uint8_t* __restrict__ scores, uint64_t n_local,
                                                         uint64_t sstride, uint32_t b, uint32_t nblocks, uint32_t shard,
                                                         uint32_t num_shards, const uint32_t* __restrict__ T,
                                                         const uint32_t* __restrict__ quota,
                                                         const uint32_t* __restrict__ base,
                                                         uint32_t* __restrict__ cands, uint64_t stride) {
    __shared__ uint32_t wg[8], wt[8];
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t blk = blockIdx.x;
    const uint64_t q = blockIdx.y;
    const uint64_t lo = uint64_t(blk) * b;
    const uint32_t len = static_cast<uint32_t>(min_u64(b, n_local - lo));
    const uint8_t* sc = scores + q * sstride + lo;
    const uint32_t t = T[q];
    const uint32_t qu = quota[q * nblocks + blk];
    uint32_t* out = cands + q * stride + base[q * nblocks + blk];
    const uint64_t gbase = lo;  // local id of the block's first point (rerank reports global ids)
    const uint32_t per = (len + blockDim.x - 1) / blockDim.x;
    const uint32_t i0 = min(len, tid * per), i1 = min(len, i0 + per);
    uint32_t g = 0, e = 0;
    for (uint32_t i = i0; i < i1; ++i) {
        const uint32_t v = sc[i];
        g += v > t;
        e += v == t;
    }
    // block exclusive scans of (g, e) in thread (= id) order
    uint32_t xg = g, xe = e;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t yg = __shfl_up_sync(kFull, xg, o), ye = __shfl_up_sync(kFull, xe, o);
        if (lane >= (uint32_t)o) {
            xg += yg;
            xe += ye;
        }
    }
    if (lane == 31) {
        wg[warp] = xg;
        wt[warp] = xe;
    }
    __syncthreads();
    uint32_t bg = 0, be = 0;
    for (uint32_t w = 0; w < warp; ++w) {
        bg += wg[w];
        be += wt[w];
    }
    uint32_t tie_rank = be + xe - e;
    uint32_t pos = bg + xg - g + min(tie_rank, qu);
    if (g + (tie_rank < qu ? e : 0u)) {
        for (uint32_t i = i0; i < i1; ++i) {
            const uint32_t v = sc[i];
            if (v > t) {
                out[pos++] = static_cast<uint32_t>(gbase + i);
            } else if (v == t && tie_rank < qu) {
                out[pos++] = static_cast<uint32_t>(gbase + i);
                ++tie_rank;
            }
        }
    }
}

// Shard construction: per (subspace, cell), how many of the cell's ids this
// shard owns, and their local ids in ascending order (cell order preserved).
__device__ __forceinline__ bool owned(uint32_t g, uint32_t b, uint32_t G, uint32_t shard) {
    return (g / b) % G == shard;
}

__global__ void shard_cell_counts_kernel(const uint32_t* __restrict__ ids, const uint32_t* __restrict__ cell_off,
                                         uint64_t n, uint32_t ns, uint32_t K, uint32_t b, uint32_t G, uint32_t shard,
                                         uint32_t* __restrict__ counts) {
    const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (t >= uint64_t(ns) * K) return;
    const uint32_t s = static_cast<uint32_t>(t / K), c = static_cast<uint32_t>(t % K);
    const uint32_t* off = cell_off + uint64_t(s) * (K + 1);
    const uint32_t* sid = ids + uint64_t(s) * n;
    uint32_t cnt = 0;
    for (uint32_t i = off[c]; i < off[c + 1]; ++i) cnt += owned(sid[i], b, G, shard);
    counts[t] = cnt;
}

__global__ void shard_compact_kernel(const uint32_t* __restrict__ ids, const uint32_t* __restrict__ cell_off, uint64_t n,
                                     uint32_t ns, uint32_t K, uint32_t b, uint32_t G, uint32_t shard,
                                     const uint32_t* __restrict__ local_off, uint64_t n_local,
                                     uint32_t* __restrict__ local_ids) {
    const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (t >= uint64_t(ns) * K) return;
    const uint32_t s = static_cast<uint32_t>(t / K), c = static_cast<uint32_t>(t % K);
    const uint32_t* off = cell_off + uint64_t(s) * (K + 1);
    const uint32_t* sid = ids + uint64_t(s) * n;
    uint32_t* out = local_ids + uint64_t(s) * n_local + local_off[uint64_t(s) * (K + 1) + c];
    for (uint32_t i = off[c]; i < off[c + 1]; ++i) {
        const uint32_t g = sid[i];
        if (owned(g, b, G, shard)) *out++ = ((g / b) / G) * b + g % b;
    }
}

__global__ void shard_ids_kernel(uint32_t* ids, uint64_t n, uint32_t b, uint32_t G, uint32_t shard) {
    const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const uint32_t l = ids[i];
    if (l != 0xffffffffu) ids[i] = ((l / b) * G + shard) * b + l % b;
}

}  // namespace

cudaError_t launch_shard_ids(uint32_t* ids, uint64_t n, uint32_t b, uint32_t G, uint32_t shard, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    shard_ids_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(ids, n, b, G, shard);
    return cudaGetLastError();
}

cudaError_t launch_shard_imi(const uint32_t* ids, const uint32_t* cell_off, uint64_t n, uint32_t ns, uint32_t K,
                             uint32_t b, uint32_t G, uint32_t shard, uint32_t* counts, const uint32_t* local_off,
                             uint64_t n_local, uint32_t* local_ids, cudaStream_t st) {
    const uint64_t total = uint64_t(ns) * K;
    const unsigned blocks = static_cast<unsigned>((total + 255) / 256);
    if (!local_ids) {
        shard_cell_counts_kernel<<<blocks, 256, 0, st>>>(ids, cell_off, n, ns, K, b, G, shard, counts);
    } else {
        shard_compact_kernel<<<blocks, 256, 0, st>>>(ids, cell_off, n, ns, K, b, G, shard, local_off, n_local, local_ids);
    }
    return cudaGetLastError();
}

cudaError_t launch_block_hist(const uint8_t* scores, uint64_t nq, uint64_t n_local, uint64_t sstride, uint32_t b,
                              uint32_t nblocks, uint32_t ns, uint32_t* hist, cudaStream_t st) {
    if (nq == 0 || nblocks == 0) return cudaSuccess;
    const bool vec = (sstride % 16 == 0) && (b % 16 == 0) && (reinterpret_cast<uintptr_t>(scores) % 16 == 0);
    if (vec && ns <= 32) {
        const dim3 grid((nblocks + 7) / 8, 1);
        for (uint64_t q0 = 0; q0 < nq; q0 += 65535) {
            const dim3 g(grid.x, static_cast<unsigned>(min_u64(65535, nq - q0)));
            const uint8_t* s0 = scores + q0 * sstride;
            uint32_t* h0 = hist + q0 * nblocks * (ns + 2);
            if (ns <= 8) block_hist_vec_kernel<8><<<g, 256, 0, st>>>(s0, n_local, sstride, b, nblocks, ns, h0);
            else if (ns <= 16) block_hist_vec_kernel<16><<<g, 256, 0, st>>>(s0, n_local, sstride, b, nblocks, ns, h0);
            else block_hist_vec_kernel<32><<<g, 256, 0, st>>>(s0, n_local, sstride, b, nblocks, ns, h0);
        }
        return cudaGetLastError();
    }
    for (uint64_t q0 = 0; q0 < nq; q0 += 65535) {
        const uint64_t nt = min_u64(65535, nq - q0);
        block_hist_kernel<<<dim3(nblocks, static_cast<unsigned>(nt)), 256, (ns + 2) * 4, st>>>(
            scores + q0 * sstride, n_local, sstride, b, nblocks, ns, hist + q0 * nblocks * (ns + 2));
    }
    return cudaGetLastError();
}

cudaError_t launch_shard_emit(const uint8_t* scores, uint64_t nq, uint64_t n_local, uint64_t sstride, uint32_t b,
                              uint32_t nblocks,
                              uint32_t shard, uint32_t num_shards, const uint32_t* T, const uint32_t* quota,
                              const uint32_t* base, uint32_t* cands, uint64_t stride, cudaStream_t st) {
    if (nq == 0 || nblocks == 0) return cudaSuccess;
    const bool vec = (sstride % 16 == 0) && (b % 16 == 0) && (reinterpret_cast<uintptr_t>(scores) % 16 == 0);
    for (uint64_t q0 = 0; q0 < nq; q0 += 65535) {
        const uint64_t nt = min_u64(65535, nq - q0);
        if (vec) {
            shard_emit_vec_kernel<<<dim3((nblocks + 7) / 8, static_cast<unsigned>(nt)), 256, 0, st>>>(
                scores + q0 * sstride, n_local, sstride, b, nblocks, shard, num_shards, T + q0, quota + q0 * nblocks,
                base + q0 * nblocks, cands + q0 * stride, stride);
            continue;
        }
        shard_emit_kernel<<<dim3(nblocks, static_cast<unsigned>(nt)), 256, 0, st>>>(
            scores + q0 * sstride, n_local, sstride, b, nblocks, shard, num_shards, T + q0, quota + q0 * nblocks,
            base + q0 * nblocks, cands + q0 * stride, stride);
    }
    return cudaGetLastError();
}

}  // namespace suco_gpu
