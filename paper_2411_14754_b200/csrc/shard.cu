// Shard-local kernels of the multi-GPU query protocol.
//
// Points are partitioned block-cyclically: with block size b and G shards,
// global block j = ids [j*b, (j+1)*b) lives on shard j % G. A shard keeps its
// blocks back to back in a local id space (local l <-> global
// ((l / b) * G + shard) * b + l % b), and keeps the GLOBAL per-cell sizes so
// that every shard's Dynamic Activation cut is the global one. The select
// plan kernels live beside the dense select they extend (dense.cu); here:
// the local IMI cut from a full one, local -> global ids, the final merge of
// every shard's local top-k, and the in-process communicator's reduction.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.h"

namespace suco_gpu {
namespace {

constexpr uint32_t kFull = 0xffffffffu;

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

// Per query (one warp): the k smallest (squared distance, id) over the G shards' local top-k
// lists — each ascending, padded with (+inf, 0xffffffff) — by a G-way merge (lane g = list g's
// head), then sqrt once (query.cpp:181-192).
__global__ void __launch_bounds__(256) merge_topk_kernel(const uint32_t* __restrict__ ids_all,
                                                         const double* __restrict__ sq_all, uint32_t G, uint64_t nq,
                                                         uint32_t k, uint32_t* __restrict__ out_ids,
                                                         double* __restrict__ out_d) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t q = uint64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (q >= nq) return;
    uint32_t head = 0;
    const uint32_t* li = ids_all + (uint64_t(lane) * nq + q) * k;
    const double* ld = sq_all + (uint64_t(lane) * nq + q) * k;
    double hd = kInf;
    uint32_t hi = 0xffffffffu;
    if (lane < G) {
        hd = ld[0];
        hi = li[0];
    }
    for (uint32_t r = 0; r < k; ++r) {
        double bd = hd;
        uint32_t bi = hi, bl = lane;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double od = __shfl_xor_sync(kFull, bd, o);
            const uint32_t oi = __shfl_xor_sync(kFull, bi, o);
            const uint32_t ol = __shfl_xor_sync(kFull, bl, o);
            if (dist_id_less(od, oi, bd, bi) || (od == bd && oi == bi && ol < bl)) {
                bd = od;
                bi = oi;
                bl = ol;
            }
        }
        if (lane == 0) {
            out_ids[q * k + r] = bi;
            out_d[q * k + r] = __dsqrt_rn(bd);
        }
        if (lane == bl && lane < G) {
            ++head;
            hd = head < k ? ld[head] : kInf;
            hi = head < k ? li[head] : 0xffffffffu;
        }
    }
}

__global__ void sum_rows_u32_kernel(const uint32_t* __restrict__ rows, uint32_t G, uint64_t count,
                                    uint32_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count; i += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t s = 0;
        for (uint32_t g = 0; g < G; ++g) s += rows[uint64_t(g) * count + i];
        out[i] = s;
    }
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

cudaError_t launch_merge_topk(const uint32_t* ids_all, const double* sq_all, uint32_t G, uint64_t nq, uint32_t k,
                              uint32_t* out_ids, double* out_d, cudaStream_t st) {
    if (nq == 0) return cudaSuccess;
    merge_topk_kernel<<<static_cast<unsigned>((nq + 7) / 8), 256, 0, st>>>(ids_all, sq_all, G, nq, k, out_ids, out_d);
    return cudaGetLastError();
}

cudaError_t launch_sum_rows_u32(const uint32_t* rows, uint32_t G, uint64_t count, uint32_t* out, cudaStream_t st) {
    if (count == 0) return cudaSuccess;
    const uint64_t blocks = min_u64((count + 255) / 256, 148ull * 8);
    sum_rows_u32_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(rows, G, count, out);
    return cudaGetLastError();
}

}  // namespace suco_gpu
