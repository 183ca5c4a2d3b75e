// SC-Linear on the GPU: the index-free baseline / quality
// oracle of sc_linear.cpp:49-121, bit-identical to it.
//
//   compute_sc_scores (sc_linear.cpp:49-93): per subspace, the exact fp64
//   squared distance of every point's whole-subspace projection to the
//   query's, then the collision_count(alpha, n) smallest by (distance, id)
//   each score one collision;
//   sc_linear_query (:95-121): the candidate_count(beta, n, k) best by
//   (score desc, id asc), re-ranked exactly.
//
// The distance follows the reference's two code paths exactly: a subspace
// whose dims are one consecutive run goes through sq_euclidean_raw (four
// strided accumulators, core.hpp:66-84); any other through
// sq_euclidean_projected (one sequential accumulator, subspace.cpp:105-121).
// Top-c per subspace is a stable radix sort of (distance bit pattern, id):
// non-negative doubles order like their bit patterns and the stable sort
// keeps ids ascending within a distance — the reference's nth_element order
// (a strict total order), so the same set. CUB's device radix sort is used
// as a library sort: this is an offline quality tool, not the query path.
#include <cub/device/device_radix_sort.cuh>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.h"

namespace suco_gpu {
namespace {

__global__ void sc_dist_kernel(ScArgs a, uint32_t s) {
    const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (i >= a.n) return;
    const float* row = a.data + i * a.d;
    {
        const uint32_t off = a.sub_off[s], len = a.sub_off[s + 1] - off;
        double dist;
        if (a.consec[s]) {  // sq_euclidean_raw over data[start, start + len)
            const float* x = row + a.dims[off];
            const float* q = a.q + a.dims[off];
            double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
            uint32_t j = 0;
            for (; j + 4 <= len; j += 4) {
                const double d0 = __dsub_rn(double(x[j]), double(q[j]));
                const double d1 = __dsub_rn(double(x[j + 1]), double(q[j + 1]));
                const double d2 = __dsub_rn(double(x[j + 2]), double(q[j + 2]));
                const double d3 = __dsub_rn(double(x[j + 3]), double(q[j + 3]));
                acc0 = __dadd_rn(acc0, __dmul_rn(d0, d0));
                acc1 = __dadd_rn(acc1, __dmul_rn(d1, d1));
                acc2 = __dadd_rn(acc2, __dmul_rn(d2, d2));
                acc3 = __dadd_rn(acc3, __dmul_rn(d3, d3));
            }
            for (; j < len; ++j) {
                const double dd = __dsub_rn(double(x[j]), double(q[j]));
                acc0 = __dadd_rn(acc0, __dmul_rn(dd, dd));
            }
            dist = __dadd_rn(__dadd_rn(acc0, acc1), __dadd_rn(acc2, acc3));
        } else {  // sq_euclidean_projected: dims in layout order, one accumulator
            double acc = 0.0;
            for (uint32_t j = 0; j < len; ++j) {
                const uint32_t dim = a.dims[off + j];
                const double dd = __dsub_rn(double(row[dim]), double(a.q[dim]));
                acc = __dadd_rn(acc, __dmul_rn(dd, dd));
            }
            dist = acc;
        }
        a.keys[i] = static_cast<unsigned long long>(__double_as_longlong(dist));
        a.vals[i] = static_cast<uint32_t>(i);
    }
}

__global__ void sc_score_kernel(const uint32_t* sorted_ids, uint64_t c, uint32_t* scores) {
    const uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (j < c) scores[sorted_ids[j]] += 1;  // the c ids are distinct: no atomics needed
}

// key = N_s - score: an ascending stable sort gives (score desc, id asc)
__global__ void sc_rank_kernel(const uint32_t* scores, uint64_t n, uint32_t ns, uint32_t* keys, uint32_t* ids) {
    const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    keys[i] = ns - scores[i];
    ids[i] = static_cast<uint32_t>(i);
}

}  // namespace

size_t sc_temp_bytes(uint64_t n) {
    size_t t1 = 0, t2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, t1, static_cast<const unsigned long long*>(nullptr),
                                    static_cast<unsigned long long*>(nullptr), static_cast<const uint32_t*>(nullptr),
                                    static_cast<uint32_t*>(nullptr), static_cast<int>(n));
    cub::DeviceRadixSort::SortPairs(nullptr, t2, static_cast<const uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                    static_cast<const uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                    static_cast<int>(n));
    return t1 > t2 ? t1 : t2;
}

cudaError_t launch_sc_scores(ScArgs a, uint64_t c, uint32_t* scores, cudaStream_t st) {
    const unsigned blocks = static_cast<unsigned>((a.n + 255) / 256);
    cudaError_t e = cudaMemsetAsync(scores, 0, a.n * 4, st);
    if (e != cudaSuccess) return e;
    for (uint32_t s = 0; s < a.ns; ++s) {  // one subspace at a time: scratch stays O(n)
        sc_dist_kernel<<<blocks, 256, 0, st>>>(a, s);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        // top-c: stable sort by distance bits keeps ids ascending within a distance
        size_t tb = a.temp_bytes;
        e = cub::DeviceRadixSort::SortPairs(a.temp, tb, a.keys, a.keys_alt, a.vals, a.vals_alt, static_cast<int>(a.n), 0,
                                            64, st);
        if (e != cudaSuccess) return e;
        sc_score_kernel<<<static_cast<unsigned>((c + 255) / 256), 256, 0, st>>>(a.vals_alt, c, scores);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t launch_sc_candidates(ScArgs a, const uint32_t* scores, uint32_t* cands_sorted, cudaStream_t st) {
    const unsigned blocks = static_cast<unsigned>((a.n + 255) / 256);
    uint32_t* keys = reinterpret_cast<uint32_t*>(a.keys);
    uint32_t* keys2 = reinterpret_cast<uint32_t*>(a.keys_alt);
    sc_rank_kernel<<<blocks, 256, 0, st>>>(scores, a.n, a.ns, keys, a.vals);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    int bits = 1;
    while ((1u << bits) <= a.ns) ++bits;
    size_t tb = a.temp_bytes;
    return cub::DeviceRadixSort::SortPairs(a.temp, tb, keys, keys2, a.vals, cands_sorted, static_cast<int>(a.n), 0, bits,
                                           st);
}

}  // namespace suco_gpu
