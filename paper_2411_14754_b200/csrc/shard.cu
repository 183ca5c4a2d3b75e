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
__global__ void block_hist_kernel(const uint8_t* __restrict__ scores, uint64_t n_local, uint32_t b, uint32_t nblocks,
                                  uint32_t ns, uint32_t* __restrict__ hist) {
    extern __shared__ uint32_t hs[];  // ns + 2
    const uint64_t q = blockIdx.y;
    const uint32_t blk = blockIdx.x;
    for (uint32_t t = threadIdx.x; t < ns + 2; t += blockDim.x) hs[t] = 0;
    __syncthreads();
    const uint64_t lo = uint64_t(blk) * b;
    const uint32_t len = static_cast<uint32_t>(min_u64(b, n_local - lo));
    const uint8_t* sc = scores + q * n_local + lo;
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

// One warp per (query, local block): emits score > T unordered-by-slot but
// block-contiguous, then the first quota ties in id order, all as GLOBAL ids,
// into cands[q][base_q_blk ...). counts[q] receives the query's total.
__global__ void shard_emit_kernel(const uint8_t* __restrict__ scores, uint64_t n_local, uint32_t b, uint32_t nblocks,
                                  uint32_t shard, uint32_t num_shards, const uint32_t* __restrict__ T,
                                  const uint32_t* __restrict__ quota, const uint32_t* __restrict__ base,
                                  uint32_t* __restrict__ cands, uint64_t stride) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t blk = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (blk >= nblocks) return;
    const uint64_t q = blockIdx.y;
    const uint64_t lo = uint64_t(blk) * b;
    const uint32_t len = static_cast<uint32_t>(min_u64(b, n_local - lo));
    const uint8_t* sc = scores + q * n_local + lo;
    const uint32_t t = T[q];
    const uint32_t qu = quota[q * nblocks + blk];
    uint32_t* out = cands + q * stride + base[q * nblocks + blk];
    const uint64_t gbase = (uint64_t(blk) * num_shards + shard) * b;  // global id of the block's first point
    uint32_t pos = 0, ties = 0;
    for (uint32_t i0 = 0; i0 < len; i0 += 32) {
        const uint32_t i = i0 + lane;
        const uint32_t v = i < len ? sc[i] : 0u;
        const bool gt = i < len && v > t;
        const bool tie = i < len && v == t;
        const uint32_t gm = __ballot_sync(kFull, gt), tm = __ballot_sync(kFull, tie);
        const uint32_t lt = (1u << lane) - 1u;
        const uint32_t tie_rank = ties + __popc(tm & lt);
        const bool take_tie = tie && tie_rank < qu;
        const uint32_t take = gm | __ballot_sync(kFull, take_tie);
        if (gt || take_tie) out[pos + __popc(take & lt)] = static_cast<uint32_t>(gbase + i);
        pos += __popc(take);
        ties += __popc(tm);
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

}  // namespace

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

cudaError_t launch_block_hist(const uint8_t* scores, uint64_t nq, uint64_t n_local, uint32_t b, uint32_t nblocks,
                              uint32_t ns, uint32_t* hist, cudaStream_t st) {
    if (nq == 0 || nblocks == 0) return cudaSuccess;
    for (uint64_t q0 = 0; q0 < nq; q0 += 65535) {
        const uint64_t nt = min_u64(65535, nq - q0);
        block_hist_kernel<<<dim3(nblocks, static_cast<unsigned>(nt)), 256, (ns + 2) * 4, st>>>(
            scores + q0 * n_local, n_local, b, nblocks, ns, hist + q0 * nblocks * (ns + 2));
    }
    return cudaGetLastError();
}

cudaError_t launch_shard_emit(const uint8_t* scores, uint64_t nq, uint64_t n_local, uint32_t b, uint32_t nblocks,
                              uint32_t shard, uint32_t num_shards, const uint32_t* T, const uint32_t* quota,
                              const uint32_t* base, uint32_t* cands, uint64_t stride, cudaStream_t st) {
    if (nq == 0 || nblocks == 0) return cudaSuccess;
    const unsigned warps_per_block = 8;
    const unsigned gx = (nblocks + warps_per_block - 1) / warps_per_block;
    for (uint64_t q0 = 0; q0 < nq; q0 += 65535) {
        const uint64_t nt = min_u64(65535, nq - q0);
        shard_emit_kernel<<<dim3(gx, static_cast<unsigned>(nt)), 32 * warps_per_block, 0, st>>>(
            scores + q0 * n_local, n_local, b, nblocks, shard, num_shards, T + q0, quota + q0 * nblocks,
            base + q0 * nblocks, cands + q0 * stride, stride);
    }
    return cudaGetLastError();
}

}  // namespace suco_gpu
