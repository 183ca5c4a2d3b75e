// Stage 1 of the query path: per-(query, subspace) centroid distances and the
// Dynamic-Activation IMI traversal, one warp per task.
//
//   centroid_distances  query.cpp:42-64   (true Euclidean, order by (dist, id))
//   dynamic_activation  query.cpp:66-121  (rows activate in rank order, argmin
//                                          over the activated prefix, ties to the
//                                          lower row; stop when cumulative >= c)
//
// Layout: the warp keeps the two ranked distance vectors (d1r/d2r), the
// rank->centroid maps and the query halves in shared memory. The DA frontier
// (one cursor per first-half rank) lives in registers, RPL rows per lane;
// each row keeps the global sizes of its next two cells prefetched, so the
// serial cumulative check rarely waits on L2.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.h"

namespace suco_gpu {
namespace {

constexpr uint32_t kFull = 0xffffffffu;

struct WarpSmem {
    double* tmp;  // k
    double* d1r;  // k
    double* d2r;  // k
    uint32_t* o1; // k
    uint32_t* o2; // k
    float* qh;    // hmax
};

__host__ __device__ inline size_t warp_smem_bytes(uint32_t k, uint32_t hmax) {
    return (size_t)k * (3 * 8 + 2 * 4) + ((hmax * 4 + 15) / 16) * 16;
}

__device__ inline WarpSmem carve(unsigned char* base, uint32_t k) {
    WarpSmem w;
    w.tmp = reinterpret_cast<double*>(base);
    w.d1r = w.tmp + k;
    w.d2r = w.d1r + k;
    w.o1 = reinterpret_cast<uint32_t*>(w.d2r + k);
    w.o2 = w.o1 + k;
    w.qh = reinterpret_cast<float*>(w.o2 + k);
    return w;
}

// Ranks `tmp` by (dist, id) (query.cpp:56-62) into dr/order; strict total order.
__device__ inline void rank_dists(const double* tmp, uint32_t k, double* dr, uint32_t* order, uint32_t lane) {
    for (uint32_t c = lane; c < k; c += 32) {
        const double dc = tmp[c];
        uint32_t r = 0;
        for (uint32_t o = 0; o < k; ++o) {
            const double dv = tmp[o];
            r += (dv < dc) || (dv == dc && o < c);
        }
        dr[r] = dc;
        order[r] = c;
    }
}

// centroid_distances for one half: dists[c] = sqrt(sq_euclidean_raw(centroid_c, q_half)).
__device__ inline void half_distances(const float* cent, const float* qh, uint32_t h, uint32_t k, double* tmp,
                                      uint32_t lane) {
    for (uint32_t c = lane; c < k; c += 32) {
        tmp[c] = __dsqrt_rn(sqdist4(cent + static_cast<size_t>(c) * h, qh, h));
    }
}

__device__ __forceinline__ uint32_t cell_sz(const uint32_t* cell_size, const uint32_t* o1, const uint32_t* o2,
                                            uint32_t k, uint32_t row, uint32_t j) {
    return j < k ? __ldg(cell_size + o1[row] * k + o2[j]) : 0u;
}

// Dynamic Activation with the frontier in registers (k <= 32 * RPL).
template <int RPL>
__device__ void da_warp(const double* d1r, const uint32_t* o1, const double* d2r, const uint32_t* o2, uint32_t k,
                        const uint32_t* cell_size, uint64_t target, uint32_t* out_cells, uint32_t* out_n,
                        double* dbg_sum, uint64_t* dbg_cum, unsigned long long* stat_cum, uint32_t lane) {
    double act[RPL];
    uint32_t cur[RPL], sz0[RPL], sz1[RPL];
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
        act[r] = kInf;
        cur[r] = 0;
        sz0[r] = 0;
        sz1[r] = 0;
    }
    if (lane == 0) {
        act[0] = __dadd_rn(d1r[0], d2r[0]);
        sz0[0] = cell_sz(cell_size, o1, o2, k, 0, 0);
        sz1[0] = cell_sz(cell_size, o1, o2, k, 0, 1);
    }
    uint32_t activated = 1, ncell = 0;
    uint64_t cum = 0;
    while (cum < target) {
        double best = act[0];
        uint32_t brow = lane;
#pragma unroll
        for (int r = 1; r < RPL; ++r) {
            if (act[r] < best) {
                best = act[r];
                brow = lane + 32u * r;
            }
        }
        // warp argmin by (distance, row): distances are >= 0, so their IEEE bit patterns order like
        // the values; three single-instruction reductions (high word, low word, row) replace a
        // five-stage shuffle butterfly on doubles
        const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(best));
        const uint32_t hi = static_cast<uint32_t>(bits >> 32), lo = static_cast<uint32_t>(bits);
        const uint32_t whi = __reduce_min_sync(kFull, hi);
        const uint32_t wlo = __reduce_min_sync(kFull, hi == whi ? lo : 0xffffffffu);
        const uint32_t pos = __reduce_min_sync(kFull, (hi == whi && lo == wlo) ? brow : 0xffffffffu);
        best = __longlong_as_double(static_cast<long long>((static_cast<uint64_t>(whi) << 32) | wlo));
        if (best == kInf) break;  // unreachable while the IMI partitions all n points
        const uint32_t owner = pos & 31u, slot = pos >> 5;
        uint32_t jm = 0, sm = 0;
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
            if (r == (int)slot) {
                jm = cur[r];
                sm = sz0[r];
            }
        }
        const uint32_t j = __shfl_sync(kFull, jm, owner);
        const uint32_t sz = __shfl_sync(kFull, sm, owner);
        cum += sz;
        if (lane == 0) {
            out_cells[ncell] = o1[pos] * k + o2[j];
            if (dbg_sum) {
                dbg_sum[ncell] = best;
                dbg_cum[ncell] = cum;
            }
        }
        ++ncell;
        if (j == 0 && activated < k) {  // query.cpp:108-112
            const uint32_t row = activated;
            if (lane == (row & 31u)) {
#pragma unroll
                for (int r = 0; r < RPL; ++r) {
                    if (r == (int)(row >> 5)) {
                        act[r] = __dadd_rn(d1r[row], d2r[0]);
                        sz0[r] = cell_sz(cell_size, o1, o2, k, row, 0);
                        sz1[r] = cell_sz(cell_size, o1, o2, k, row, 1);
                    }
                }
            }
            ++activated;
        }
        if (lane == owner) {  // query.cpp:113-118
#pragma unroll
            for (int r = 0; r < RPL; ++r) {
                if (r == (int)slot) {
                    if (j + 1 == k) {
                        act[r] = kInf;
                    } else {
                        cur[r] = j + 1;
                        act[r] = __dadd_rn(d1r[pos], d2r[j + 1]);
                        sz0[r] = sz1[r];
                        sz1[r] = cell_sz(cell_size, o1, o2, k, pos, j + 2);
                    }
                }
            }
        }
    }
    if (lane == 0) {
        *out_n = ncell;
        if (stat_cum) atomicAdd(stat_cum, static_cast<unsigned long long>(cum));
    }
}

// k <= 64 (two rows per lane: lane and lane + 32): the frontier of both rows in named registers
// (the generic RPL arrays ended up in local memory), updated by selects.
__device__ void da_warp2(const double* d1r, const uint32_t* o1, const double* d2r, const uint32_t* o2, uint32_t k,
                         const uint32_t* cell_size, uint64_t target, uint32_t* out_cells, uint32_t* out_n,
                         double* dbg_sum, uint64_t* dbg_cum, unsigned long long* stat_cum, uint32_t lane) {
    double a0 = kInf, a1 = kInf;          // next sum of row lane / row lane + 32
    uint32_t c0 = 0, c1 = 0;              // their cursors (second-half rank)
    uint32_t s00 = 0, s01 = 0, s10 = 0, s11 = 0;  // sizes of each row's next two cells
    if (lane == 0) {
        a0 = __dadd_rn(d1r[0], d2r[0]);
        s00 = cell_sz(cell_size, o1, o2, k, 0, 0);
        s01 = cell_sz(cell_size, o1, o2, k, 0, 1);
    }
    uint32_t activated = 1, ncell = 0;
    uint64_t cum = 0;
    while (cum < target) {
        const bool second = a1 < a0;  // ties keep the lower row (lane < lane + 32)
        const double best = second ? a1 : a0;
        const uint32_t brow = second ? lane + 32u : lane;
        // warp argmin by (distance, row) on the non-negative distances' bit patterns
        const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(best));
        const uint32_t hi = static_cast<uint32_t>(bits >> 32), lo = static_cast<uint32_t>(bits);
        const uint32_t whi = __reduce_min_sync(kFull, hi);
        const uint32_t wlo = __reduce_min_sync(kFull, hi == whi ? lo : 0xffffffffu);
        const uint32_t pos = __reduce_min_sync(kFull, (hi == whi && lo == wlo) ? brow : 0xffffffffu);
        if (whi >= 0x7ff00000u) break;  // +inf: unreachable while the IMI partitions all n points
        const uint32_t owner = pos & 31u;
        const bool slot1 = pos >= 32u;
        const uint32_t j = __shfl_sync(kFull, slot1 ? c1 : c0, owner);
        const uint32_t sz = __shfl_sync(kFull, slot1 ? s10 : s00, owner);
        cum += sz;
        if (lane == 0) {
            out_cells[ncell] = o1[pos] * k + o2[j];
            if (dbg_sum) {
                dbg_sum[ncell] = __longlong_as_double(static_cast<long long>((static_cast<uint64_t>(whi) << 32) | wlo));
                dbg_cum[ncell] = cum;
            }
        }
        ++ncell;
        if (j == 0 && activated < k) {  // query.cpp:108-112: the next row joins the frontier
            const uint32_t row = activated;
            if (lane == (row & 31u)) {
                const double v = __dadd_rn(d1r[row], d2r[0]);
                const uint32_t z0 = cell_sz(cell_size, o1, o2, k, row, 0), z1 = cell_sz(cell_size, o1, o2, k, row, 1);
                if (row >= 32u) {
                    a1 = v;
                    s10 = z0;
                    s11 = z1;
                } else {
                    a0 = v;
                    s00 = z0;
                    s01 = z1;
                }
            }
            ++activated;
        }
        if (lane == owner) {  // query.cpp:113-118: advance the retrieved row
            const bool done = j + 1 == k;
            const double v = done ? kInf : __dadd_rn(d1r[pos], d2r[j + 1]);
            const uint32_t z = done ? 0u : cell_sz(cell_size, o1, o2, k, pos, j + 2);
            if (slot1) {
                c1 = j + 1;
                a1 = v;
                s10 = s11;
                s11 = z;
            } else {
                c0 = j + 1;
                a0 = v;
                s00 = s01;
                s01 = z;
            }
        }
    }
    if (lane == 0) {
        *out_n = ncell;
        if (stat_cum) atomicAdd(stat_cum, static_cast<unsigned long long>(cum));
    }
}

// Frontier in shared memory for k > 256 (rare: large k_half traversal tests).
__device__ void da_warp_smem(const double* d1r, const uint32_t* o1, const double* d2r, const uint32_t* o2, uint32_t k,
                             const uint32_t* cell_size, uint64_t target, uint32_t* out_cells, uint32_t* out_n,
                             double* dbg_sum, uint64_t* dbg_cum, unsigned long long* stat_cum, uint32_t lane,
                             double* act, uint32_t* cur) {
    for (uint32_t r = lane; r < k; r += 32) {
        act[r] = kInf;
        cur[r] = 0;
    }
    __syncwarp();
    if (lane == 0) act[0] = __dadd_rn(d1r[0], d2r[0]);
    __syncwarp();
    uint32_t activated = 1, ncell = 0;
    uint64_t cum = 0;
    while (cum < target) {
        double best = kInf;
        uint32_t brow = 0xffffffffu;
        for (uint32_t r = lane; r < activated; r += 32) {
            const double v = act[r];
            if (v < best) {
                best = v;
                brow = r;
            }
        }
        for (int off = 16; off > 0; off >>= 1) {
            const double ob = __shfl_xor_sync(kFull, best, off);
            const uint32_t orow = __shfl_xor_sync(kFull, brow, off);
            if (ob < best || (ob == best && orow < brow)) {
                best = ob;
                brow = orow;
            }
        }
        if (best == kInf) break;
        const uint32_t pos = brow;
        const uint32_t j = cur[pos];
        cum += __ldg(cell_size + o1[pos] * k + o2[j]);
        if (lane == 0) {
            out_cells[ncell] = o1[pos] * k + o2[j];
            if (dbg_sum) {
                dbg_sum[ncell] = best;
                dbg_cum[ncell] = cum;
            }
        }
        ++ncell;
        __syncwarp();
        if (lane == 0) {
            if (j == 0 && activated < k) act[activated] = __dadd_rn(d1r[activated], d2r[0]);
            if (j + 1 == k) {
                act[pos] = kInf;
            } else {
                cur[pos] = j + 1;
                act[pos] = __dadd_rn(d1r[pos], d2r[j + 1]);
            }
        }
        if (j == 0 && activated < k) ++activated;
        __syncwarp();
    }
    if (lane == 0) {
        *out_n = ncell;
        if (stat_cum) atomicAdd(stat_cum, static_cast<unsigned long long>(cum));
    }
}

__device__ inline void run_da(const WarpSmem& w, uint32_t k, const uint32_t* cell_size, uint64_t target,
                              uint32_t* out_cells, uint32_t* out_n, double* dbg_sum, uint64_t* dbg_cum,
                              unsigned long long* stat_cum, uint32_t lane) {
    if (k <= 64) {
        da_warp2(w.d1r, w.o1, w.d2r, w.o2, k, cell_size, target, out_cells, out_n, dbg_sum, dbg_cum, stat_cum, lane);
    } else if (k <= 128) {
        da_warp<4>(w.d1r, w.o1, w.d2r, w.o2, k, cell_size, target, out_cells, out_n, dbg_sum, dbg_cum, stat_cum,
                    lane);
    } else if (k <= 256) {
        da_warp<8>(w.d1r, w.o1, w.d2r, w.o2, k, cell_size, target, out_cells, out_n, dbg_sum, dbg_cum, stat_cum,
                    lane);
    } else {
        // the tmp array (k doubles) is free after ranking: reuse it as the
        // frontier distances, and the query-half area is too small for the
        // cursors, so the caller provides k extra u32 after the warp block.
        da_warp_smem(w.d1r, w.o1, w.d2r, w.o2, k, cell_size, target, out_cells, out_n, dbg_sum, dbg_cum, stat_cum,
                     lane, w.tmp, reinterpret_cast<uint32_t*>(w.qh));
    }
}

__global__ void __launch_bounds__(256, 5) traverse_kernel(TraverseArgs a, uint32_t warps_per_block, size_t per_warp) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint64_t task = static_cast<uint64_t>(blockIdx.x) * warps_per_block + warp;
    if (task >= a.nq * a.ns) return;
    const uint64_t q = task / a.ns;
    const uint32_t s = static_cast<uint32_t>(task % a.ns);
    const uint32_t k = a.k_half;
    WarpSmem w = carve(smem + per_warp * warp, k);
    const SubDesc sd = a.sub[s];
    const float* query = a.queries + q * a.d;

    // first half: project (subspace.cpp:83-92), distances, rank
    for (uint32_t i = lane; i < sd.h1; i += 32) w.qh[i] = query[a.dims[sd.dims1 + i]];
    __syncwarp();
    half_distances(a.cent + sd.cent1, w.qh, sd.h1, k, w.tmp, lane);
    __syncwarp();
    rank_dists(w.tmp, k, w.d1r, w.o1, lane);
    __syncwarp();
    // second half
    for (uint32_t i = lane; i < sd.h2; i += 32) w.qh[i] = query[a.dims[sd.dims2 + i]];
    __syncwarp();
    half_distances(a.cent + sd.cent2, w.qh, sd.h2, k, w.tmp, lane);
    __syncwarp();
    rank_dists(w.tmp, k, w.d2r, w.o2, lane);
    __syncwarp();

    const uint64_t t = q * a.ns + s;
    run_da(w, k, a.cell_size + static_cast<size_t>(s) * a.K, a.target, a.cells + t * a.K, a.ncells + t,
           a.dbg_sum ? a.dbg_sum + t * a.K : nullptr, a.dbg_cum ? a.dbg_cum + t * a.K : nullptr, a.stat_cum, lane);
}

__global__ void centroid_distances_kernel(const float* q, uint32_t dim, const float* cent, uint32_t k,
                                          double* dists, uint32_t* order) {
    extern __shared__ __align__(16) unsigned char smem[];
    double* tmp = reinterpret_cast<double*>(smem);
    const uint32_t lane = threadIdx.x & 31u;
    half_distances(cent, q, dim, k, tmp, lane);
    __syncwarp();
    for (uint32_t c = lane; c < k; c += 32) dists[c] = tmp[c];
    double* dr = tmp + k;
    rank_dists(tmp, k, dr, order, lane);
}

__global__ void da_only_kernel(const double* d1, const uint32_t* o1, const double* d2, const uint32_t* o2,
                               uint32_t k, const uint32_t* cell_size, uint64_t target, uint32_t* cells,
                               uint32_t* ncells, double* sums, uint64_t* cum) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t lane = threadIdx.x & 31u;
    WarpSmem w = carve(smem, k);
    for (uint32_t i = lane; i < k; i += 32) {
        w.o1[i] = o1[i];
        w.o2[i] = o2[i];
        w.d1r[i] = d1[o1[i]];  // ranked(): query.cpp:34-38
        w.d2r[i] = d2[o2[i]];
    }
    __syncwarp();
    run_da(w, k, cell_size, target, cells, ncells, sums, cum, nullptr, lane);
}

}  // namespace

static size_t da_extra_bytes(uint32_t k) { return k > 256 ? static_cast<size_t>(k) * 4 + 16 : 0; }

cudaError_t launch_traverse(const TraverseArgs& a, cudaStream_t st) {
    if (a.nq == 0) return cudaSuccess;
    const size_t per_warp = ((warp_smem_bytes(a.k_half, a.hmax) + da_extra_bytes(a.k_half) + 15) / 16) * 16;
    uint32_t wpb = static_cast<uint32_t>(48 * 1024 / per_warp);
    if (wpb > 8) wpb = 8;
    if (wpb < 1) wpb = 1;
    const size_t smem = per_warp * wpb;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(traverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    const uint64_t tasks = a.nq * a.ns;
    const uint64_t blocks = (tasks + wpb - 1) / wpb;
    traverse_kernel<<<static_cast<unsigned>(blocks), 32 * wpb, smem, st>>>(a, wpb, per_warp);
    return cudaGetLastError();
}

cudaError_t launch_centroid_distances(const float* d_q, uint32_t dim, const float* d_cent, uint32_t k_half,
                                      double* d_dists, uint32_t* d_order, cudaStream_t st) {
    const size_t smem = static_cast<size_t>(k_half) * 16;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(centroid_distances_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    centroid_distances_kernel<<<1, 32, smem, st>>>(d_q, dim, d_cent, k_half, d_dists, d_order);
    return cudaGetLastError();
}

cudaError_t launch_da_only(const double* d1, const uint32_t* o1, const double* d2, const uint32_t* o2,
                           uint32_t k_half, const uint32_t* cell_size, uint64_t target, uint32_t* cells,
                           uint32_t* ncells, double* sums, uint64_t* cum, cudaStream_t st) {
    const size_t smem = ((warp_smem_bytes(k_half, 1) + da_extra_bytes(k_half) + 15) / 16) * 16;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(da_only_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    da_only_kernel<<<1, 32, smem, st>>>(d1, o1, d2, o2, k_half, cell_size, target, cells, ncells, sums, cum);
    return cudaGetLastError();
}

}  // namespace suco_gpu
