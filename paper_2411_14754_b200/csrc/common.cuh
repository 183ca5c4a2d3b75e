// Shared device helpers and the device-resident index layout.
//
// Exactness contract (SURVEY §7 hard part 1): every distance on the path is
// the reference's fp64 kernel sq_euclidean_raw (core.hpp:66-84) — per-dim
// (double)a - (double)b, squared, folded into four strided accumulators in
// index order with the tail in acc0, combined (a0+a1)+(a2+a3). On the device
// each op is an explicit round-to-nearest intrinsic (__dsub_rn/__dmul_rn/
// __dadd_rn) and the library is compiled with -fmad=false, so no DFMA can
// contract a product into a sum. sqrt is __dsqrt_rn (IEEE, like std::sqrt).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#ifndef SUCO_HD
#define SUCO_HD __host__ __device__ __forceinline__
#endif

namespace suco_gpu {

constexpr double kInf = __builtin_huge_val();

SUCO_HD uint64_t min_u64(uint64_t a, uint64_t b) { return a < b ? a : b; }

// (d_a - d_b)^2 with IEEE double rounding at every step.
__device__ __forceinline__ double sqdiff(float a, float b) {
    const double d = __dsub_rn(static_cast<double>(a), static_cast<double>(b));
    return __dmul_rn(d, d);
}

__device__ __forceinline__ double sqdiff_d(float a, double b) {
    const double d = __dsub_rn(static_cast<double>(a), b);
    return __dmul_rn(d, d);
}

// core.hpp:66-84 restated for contiguous spans (a: first operand, b: second).
__device__ __forceinline__ double sqdist4(const float* a, const float* b, uint32_t len) {
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
    uint32_t i = 0;
    for (; i + 4 <= len; i += 4) {
        acc0 = __dadd_rn(acc0, sqdiff(a[i], b[i]));
        acc1 = __dadd_rn(acc1, sqdiff(a[i + 1], b[i + 1]));
        acc2 = __dadd_rn(acc2, sqdiff(a[i + 2], b[i + 2]));
        acc3 = __dadd_rn(acc3, sqdiff(a[i + 3], b[i + 3]));
    }
    for (; i < len; ++i) acc0 = __dadd_rn(acc0, sqdiff(a[i], b[i]));
    return __dadd_rn(__dadd_rn(acc0, acc1), __dadd_rn(acc2, acc3));
}

// Per-subspace descriptor: half dims, offsets of each half's dimension list
// in the concatenated dims array and of each half's centroids in the
// concatenated centroid array.
struct SubDesc {
    uint32_t h1, h2;
    uint32_t dims1, dims2;
    uint64_t cent1, cent2;
};

// Lexicographic (dist, id) order used by rerank's top-k (query.cpp:181-186).
__device__ __forceinline__ bool dist_id_less(double da, uint32_t ia, double db, uint32_t ib) {
    return da < db || (da == db && ia < ib);
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

}  // namespace suco_gpu
