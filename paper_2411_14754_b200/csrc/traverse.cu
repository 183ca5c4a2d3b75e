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

#include <cstdlib>
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

// ---------------------------------------------------------------------------
// Two-phase traversal (default for 6 <= k_half <= 128). The centroid distances and the O(k^2)
// (dist, id) ranking are most of a task's instructions, and in the thread-per-task kernel they run
// at the merge's occupancy (a few warps per SM: ~1.8 KB of merge state per task). Phase 1 ranks
// every (query, subspace, half) with one WARP each — no per-thread state, full occupancy — and
// leaves the ranked distances and rank -> centroid maps in a record at the tail of the task's own
// row of the cell-list output (K words per task, of which Dynamic Activation fills ~alpha * K from
// the front, and only after phase 2 has copied the record into shared memory). Phase 2 is the
// thread-per-task merge alone.
//
// Record of task t (16-byte aligned, inside cells[t*K .. (t+1)*K)): d1r[k], d2r[k] (f64), o1[k],
// o2[k] (u8).
__host__ __device__ inline bool rank_rec_fits(uint32_t k, uint32_t K) { return 4ull * K >= 18ull * k + 16ull && k >= 2; }

__device__ __forceinline__ unsigned char* rank_rec(uint32_t* cells, uint64_t task, uint32_t K, uint32_t k) {
    const uintptr_t end = reinterpret_cast<uintptr_t>(cells + (task + 1) * K);
    return reinterpret_cast<unsigned char*>((end - 18u * k) & ~static_cast<uintptr_t>(15));
}

// rank of c = #{o : (d_o, o) < (d_c, c)} for the U elements c = lane + 32u of one lane, in one pass
// over o: every loaded value serves U independent counters. Without ties the rank is #{o : d_o <
// d_c} — one comparison per pair. Tied elements count the same number of strictly smaller values and
// collide in a shared-memory scatter of their ids, which the owners see when they read it back; only then the warp
// ranks again with the id tie-break (query.cpp:56-62).
template <uint32_t U>
__device__ __forceinline__ void rank_warp(const double* scr, uint8_t* slot, uint32_t k, double* dr, uint8_t* ord,
                                          uint32_t lane) {
    double dc[U];
    uint32_t r[U];
#pragma unroll
    for (uint32_t u = 0; u < U; ++u) {
        const uint32_t c = lane + 32u * u;
        dc[u] = c < k ? scr[c] : kInf;
        r[u] = 0;
    }
#pragma unroll 8
    for (uint32_t o = 0; o < k; ++o) {
        const double v = scr[o];
#pragma unroll
        for (uint32_t u = 0; u < U; ++u) r[u] += v < dc[u];
    }
#pragma unroll
    for (uint32_t u = 0; u < U; ++u) {
        const uint32_t c = lane + 32u * u;
        if (c < k) slot[r[u]] = static_cast<uint8_t>(c);
    }
    __syncwarp();
    bool lost = false;
#pragma unroll
    for (uint32_t u = 0; u < U; ++u) {
        const uint32_t c = lane + 32u * u;
        if (c < k) {
            lost |= slot[r[u]] != static_cast<uint8_t>(c);
            dr[r[u]] = dc[u];
            ord[r[u]] = static_cast<uint8_t>(c);
        }
    }
    if (__any_sync(kFull, lost)) {  // ties: exact (dist, id) ranks
        __syncwarp();
#pragma unroll 1
        for (uint32_t u = 0; u < U; ++u) {
            const uint32_t c = lane + 32u * u;
            if (c >= k) continue;
            const double d = scr[c];
            uint32_t rr = 0;
            for (uint32_t o = 0; o < k; ++o) {
                const double v = scr[o];
                rr += v < d || (v == d && o < c);
            }
            dr[rr] = d;
            ord[rr] = static_cast<uint8_t>(c);
        }
    }
}

constexpr uint32_t kRankWarps = 8;

// grid (ceil(nq / kRankWarps), 2 * ns): one warp per (query, subspace, half).
template <uint32_t U>
__global__ void __launch_bounds__(32 * kRankWarps) rank_halves_kernel(TraverseArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint32_t s = blockIdx.y >> 1, half = blockIdx.y & 1u, k = a.k_half;
    const uint64_t q = static_cast<uint64_t>(blockIdx.x) * kRankWarps + warp;
    if (q >= a.nq) return;
    double* scr = reinterpret_cast<double*>(smem) + static_cast<size_t>(warp) * k;
    float* qh = reinterpret_cast<float*>(reinterpret_cast<double*>(smem) + static_cast<size_t>(kRankWarps) * k) +
                static_cast<size_t>(warp) * a.hmax;
    uint8_t* slot = reinterpret_cast<uint8_t*>(reinterpret_cast<double*>(smem) + static_cast<size_t>(kRankWarps) * k) +
                    static_cast<size_t>(kRankWarps) * a.hmax * 4 + static_cast<size_t>(warp) * 128;
    const SubDesc sd = a.sub[s];
    const uint32_t h = half ? sd.h2 : sd.h1;
    const uint32_t* dims = a.dims + (half ? sd.dims2 : sd.dims1);
    const float* query = a.queries + q * a.d;
    for (uint32_t i = lane; i < h; i += 32) qh[i] = query[__ldg(dims + i)];  // project_into (subspace.cpp:83-92)
    __syncwarp();
    half_distances(a.cent + (half ? sd.cent2 : sd.cent1), qh, h, k, scr, lane);  // query.cpp:42-55
    __syncwarp();
    unsigned char* rec = rank_rec(a.cells, q * a.ns + s, a.K, k);
    rank_warp<U>(scr, slot, k, reinterpret_cast<double*>(rec) + (half ? k : 0u), rec + 16u * k + (half ? k : 0u), lane);
}

// (ka, ra) < (kb, rb) lexicographically on the BIT PATTERNS of non-negative doubles (their integer
// order is their numeric order, +inf above every finite value): the borrow of one 96-bit
// subtraction — four dependent integer adds instead of two dependent FP64 compares, whose latency
// is what a pop of the merge waits on (one warp per scheduler, nothing to hide it).
__device__ __forceinline__ bool key_row_less(uint64_t ka, uint32_t ra, uint64_t kb, uint32_t rb) {
    uint32_t borrow;
    asm("{\n\t.reg .u32 t;\n\tsub.cc.u32 t, %1, %2;\n\tsubc.cc.u32 t, %3, %4;\n\tsubc.cc.u32 t, %5, %6;\n\tsubc.u32 %0, 0, 0;\n\t}"
        : "=r"(borrow)
        : "r"(ra), "r"(rb), "r"(static_cast<uint32_t>(ka)), "r"(static_cast<uint32_t>(kb)),
          "r"(static_cast<uint32_t>(ka >> 32)), "r"(static_cast<uint32_t>(kb >> 32)));
    return borrow != 0;
}

// ---------------------------------------------------------------------------
// Thread-per-task traversal (k_half <= 128): one thread owns one (query,
// subspace) task end to end; a CTA holds tasks of ONE subspace, so that
// subspace's cell sizes sit in shared memory and the cumulative check never
// waits on L2.
//
// Dynamic Activation is the k-way merge of the k rows (row r = cells
// (r, 0..k-1) in second-half rank order) by (d1r[r] + d2r[j], r): an
// unactivated row r's head (r, 0) never beats row r-1's, which is still at
// (r-1, 0) while r is unactivated (d1r ascending, rounding monotone, ties to
// the lower row) — so merging all rows from the start pops exactly the
// reference's sequence (query.cpp:66-121), and the debug outputs match too.
// The merge is a loser tree over L >= k leaves: the initial heads are already
// in (key, row) order, so every node's loser is the leftmost leaf of its right
// subtree (closed form, no comparisons). A pop replays one leaf-to-root path
// whose nodes depend only on the row, so all its loads issue at once.
//
// Per-thread arrays are interleaved [element][thread]: threads reading the
// same element index hit consecutive words.
// SPLIT: two threads per task (adjacent lanes) compute and rank one half each — the centroid
// distances and the O(k^2) ranking are most of a task's latency — then the even thread runs
// Dynamic Activation alone; each half has its own ranking scratch and projected query.
// PRE: the halves arrive ranked (rank_halves_kernel's records); the thread only merges.
template <uint32_t L, uint32_t SP, bool PRE = false>  // SP threads per task: 1, 2 (one half each) or 4 (half a half each)
__global__ void traverse_thread_kernel(TraverseArgs a) {
    static_assert(!PRE || SP == 1, "pre-ranked halves: one thread per task");
    constexpr bool SPLIT = SP > 1;
    constexpr uint32_t LOG = L == 64 ? 6 : 7;
    static_assert(L == 64 || L == 128, "leaves");
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t T = blockDim.x / SP, t = threadIdx.x / SP;
    const uint32_t s = blockIdx.y, k = a.k_half, K = a.K;
    double* tkey = reinterpret_cast<double*>(smem);  // [L][T]: loser keys (nodes 1..L-1); ranking scratch
    double* d1r = tkey + L * T;                       // [k][T]
    double* d2r = d1r + k * T;                        // [k][T]
    double* scr2 = d2r + k * T;                       // SPLIT: [k][T] the second half's ranking scratch
    uint32_t* cs = reinterpret_cast<uint32_t*>(scr2 + (SPLIT ? k * T : 0));  // [K] this subspace's cell sizes
    // PRE with cs_global: the cell sizes stay in global memory (L2; the cumulative check is off the
    // merge's critical path) and their K words of shared memory go to more resident tasks
    const bool csg = PRE && a.cs_global != 0;
    const uint32_t* csz = a.cell_size + static_cast<size_t>(s) * K;
    float* qh = reinterpret_cast<float*>(cs + (csg ? 0u : K));  // [hmax][T] (x2 with SPLIT; none with PRE)
    uint8_t* trow = reinterpret_cast<uint8_t*>(qh + (PRE ? 0u : a.hmax * T * (SPLIT ? 2 : 1)));  // [L][T]
    uint8_t* o1 = trow + L * T;  // [k][T]
    uint8_t* o2 = o1 + k * T;
    uint8_t* cur = o2 + k * T;
    const uint64_t q = static_cast<uint64_t>(blockIdx.x) * T + t;
    if (!csg) {
#pragma unroll 8
        for (uint32_t i = threadIdx.x; i < K; i += blockDim.x) cs[i] = __ldg(csz + i);
    }
    __syncthreads();
    if (q >= a.nq) return;
    const SubDesc sd = a.sub[s];
    const float* query = a.queries + q * a.d;

    // centroid_distances (query.cpp:42-64) for both halves, ranked by (dist, id)
    const uint32_t sub = threadIdx.x % SP;
    const uint32_t h_lo = SP == 4 ? sub >> 1 : SP == 2 ? sub : 0u, h_hi = SPLIT ? h_lo + 1 : 2u;
    // SP = 4: the two threads of a half split its k centroids (distances, then ranks)
    const uint32_t kpart = (a.k_half + 1) / 2;
    const uint32_t c_lo = SP == 4 ? (sub & 1u) * kpart : 0u, c_hi = SP == 4 ? min(a.k_half, c_lo + kpart) : a.k_half;
    const uint32_t lane = threadIdx.x & 31u;
    if constexpr (PRE) {
        // the task's record: 16-byte loads of the ranked distances, then the rank -> centroid bytes
        const unsigned char* rec = rank_rec(a.cells, q * a.ns + s, K, k);
        const double2* rd = reinterpret_cast<const double2*>(rec);
#pragma unroll 8
        for (uint32_t e = 0; e < k; ++e) {  // 2k doubles = k double2: d1r[0..k) then d2r[0..k)
            const double2 v = rd[e];
            const uint32_t e0 = 2 * e, e1 = 2 * e + 1;
            (e0 < k ? d1r[e0 * T + t] : d2r[(e0 - k) * T + t]) = v.x;
            (e1 < k ? d1r[e1 * T + t] : d2r[(e1 - k) * T + t]) = v.y;
        }
        const unsigned char* ro = rec + 16u * k;
        if ((k & 1u) == 0) {
            const uint16_t* r2 = reinterpret_cast<const uint16_t*>(ro);
            for (uint32_t e = 0; e < k; e += 2) {
                const uint32_t v1 = r2[e >> 1], v2 = r2[(k + e) >> 1];
                o1[e * T + t] = static_cast<uint8_t>(v1);
                o1[(e + 1) * T + t] = static_cast<uint8_t>(v1 >> 8);
                o2[e * T + t] = static_cast<uint8_t>(v2);
                o2[(e + 1) * T + t] = static_cast<uint8_t>(v2 >> 8);
            }
        } else {
            for (uint32_t e = 0; e < k; ++e) {
                o1[e * T + t] = ro[e];
                o2[e * T + t] = ro[k + e];
            }
        }
        // (the record sits in the tail of this task's own cell row: it is in shared memory before
        // the merge below writes the row's first cell)
    }
#pragma unroll 1
    for (uint32_t half = PRE ? 2u : h_lo; half < h_hi; ++half) {
        const uint32_t h = half ? sd.h2 : sd.h1;
        const uint32_t* dims = a.dims + (half ? sd.dims2 : sd.dims1);
        const float* cent = a.cent + (half ? sd.cent2 : sd.cent1);
        double* dr = half ? d2r : d1r;
        uint8_t* ord = half ? o2 : o1;
        double* scr = SPLIT && half ? scr2 : tkey;  // ranking scratch of this half
        float* qp = SPLIT && half ? qh + a.hmax * T : qh;
        if (SP < 4 || (sub & 1u) == 0) {
            for (uint32_t i = 0; i < h; ++i) qp[i * T + t] = query[__ldg(dims + i)];
        }
        if constexpr (SP == 4) __syncwarp(3u << (lane & ~1u));  // the half's projected query
        for (uint32_t c = c_lo; c < c_hi; ++c) {  // sq_euclidean_raw (core.hpp:66-84) then sqrt
            const float* cc = cent + static_cast<size_t>(c) * h;
            double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
            uint32_t i = 0;
            for (; i + 4 <= h; i += 4) {
                acc0 = __dadd_rn(acc0, sqdiff(__ldg(cc + i), qp[i * T + t]));
                acc1 = __dadd_rn(acc1, sqdiff(__ldg(cc + i + 1), qp[(i + 1) * T + t]));
                acc2 = __dadd_rn(acc2, sqdiff(__ldg(cc + i + 2), qp[(i + 2) * T + t]));
                acc3 = __dadd_rn(acc3, sqdiff(__ldg(cc + i + 3), qp[(i + 3) * T + t]));
            }
            for (; i < h; ++i) acc0 = __dadd_rn(acc0, sqdiff(__ldg(cc + i), qp[i * T + t]));
            scr[c * T + t] = __dsqrt_rn(__dadd_rn(__dadd_rn(acc0, acc1), __dadd_rn(acc2, acc3)));
        }
        if constexpr (SP == 4) __syncwarp(3u << (lane & ~1u));  // every distance of the half
        // rank of c = #{o : (d_o, o) < (d_c, c)}; four c per pass over o, the id tie-break folded
        // into the loop bounds (o < c0: <=, o >= c0 + 4: <, the group itself: exact)
        for (uint32_t c0 = c_lo; c0 < c_hi; c0 += 4) {
            double dc[4];
            uint32_t r[4];
#pragma unroll
            for (uint32_t u = 0; u < 4; ++u) {
                dc[u] = c0 + u < c_hi ? scr[(c0 + u) * T + t] : kInf;
                r[u] = 0;
            }
            for (uint32_t o = 0; o < c0; ++o) {
                const double v = scr[o * T + t];
#pragma unroll
                for (uint32_t u = 0; u < 4; ++u) r[u] += v <= dc[u];
            }
            for (uint32_t o = c0; o < c0 + 4 && o < k; ++o) {
                const double v = scr[o * T + t];
#pragma unroll
                for (uint32_t u = 0; u < 4; ++u) r[u] += v < dc[u] || (v == dc[u] && o < c0 + u);
            }
            // (group members past c_hi are padding: kInf never counts against real values, and their
            // own ranks are not stored)
            for (uint32_t o = c0 + 4; o < k; ++o) {
                const double v = scr[o * T + t];
#pragma unroll
                for (uint32_t u = 0; u < 4; ++u) r[u] += v < dc[u];
            }
#pragma unroll
            for (uint32_t u = 0; u < 4; ++u) {
                if (c0 + u < c_hi) {
                    dr[r[u] * T + t] = dc[u];
                    ord[r[u] * T + t] = static_cast<uint8_t>(c0 + u);
                }
            }
        }
    }

    if constexpr (SPLIT) {  // the task's other parts are in shared memory; thread 0 of the task goes on
        __syncwarp(((1u << SP) - 1u) << (lane & ~(SP - 1u)));
        if (sub != 0) return;
    }
    // loser tree over the row heads (r, 0): node n at level lv loses with the leftmost leaf of its
    // right child
    const double d20 = d2r[t];
    for (uint32_t lv = 0; lv < LOG; ++lv) {
        for (uint32_t n = 1u << lv; n < (2u << lv); ++n) {
            const uint32_t leaf = ((2 * n + 1) << (LOG - lv - 1)) - L;
            tkey[n * T + t] = leaf < k ? __dadd_rn(d1r[leaf * T + t], d20) : kInf;
            trow[n * T + t] = static_cast<uint8_t>(leaf);
        }
    }
    for (uint32_t r = 0; r < k; ++r) cur[r * T + t] = 0;
    constexpr uint64_t kInfBits = 0x7ff0000000000000ull;
    uint64_t* tbits = reinterpret_cast<uint64_t*>(tkey);  // the tree's keys, compared as integers
    uint64_t wkey = static_cast<uint64_t>(__double_as_longlong(__dadd_rn(d1r[t], d20)));
    uint32_t wrow = 0;

    const uint64_t task = q * a.ns + s;
    uint32_t* out = a.cells + task * K;
    double* dbg_sum = a.dbg_sum ? a.dbg_sum + task * K : nullptr;
    uint64_t* dbg_cum = a.dbg_cum ? a.dbg_cum + task * K : nullptr;
    uint32_t ncell = 0;
    uint64_t cum = 0;
    while (cum < a.target) {
        if (wkey == kInfBits) break;  // unreachable while the IMI partitions all n points
        const uint32_t row = wrow, j = cur[row * T + t];
        const uint32_t cell = static_cast<uint32_t>(o1[row * T + t]) * k + o2[j * T + t];
        cum += csg ? __ldg(csz + cell) : cs[cell];
        out[ncell] = cell;
        if (dbg_sum) {
            dbg_sum[ncell] = __longlong_as_double(static_cast<long long>(wkey));
            dbg_cum[ncell] = cum;
        }
        ++ncell;
        // the row's next cell (query.cpp:113-118), then replay its leaf-to-root path
        const uint32_t j1 = j + 1;
        cur[row * T + t] = static_cast<uint8_t>(j1);
        uint64_t ck = j1 < k ? static_cast<uint64_t>(__double_as_longlong(__dadd_rn(d1r[row * T + t], d2r[j1 * T + t])))
                             : kInfBits;
        uint32_t cr = row;
        const uint32_t n0 = (row + L) >> 1;
        uint64_t pk[LOG];
        uint32_t pr[LOG];
#pragma unroll
        for (uint32_t lv = 0; lv < LOG; ++lv) {
            pk[lv] = tbits[(n0 >> lv) * T + t];
            pr[lv] = trow[(n0 >> lv) * T + t];
        }
#pragma unroll
        for (uint32_t lv = 0; lv < LOG; ++lv) {
            if (key_row_less(pk[lv], pr[lv], ck, cr)) {  // the stored loser wins: swap
                const uint32_t n = n0 >> lv;
                tbits[n * T + t] = ck;
                trow[n * T + t] = static_cast<uint8_t>(cr);
                ck = pk[lv];
                cr = pr[lv];
            }
        }
        wkey = ck;
        wrow = cr;
    }
    a.ncells[task] = ncell;
    if (a.stat_cum) atomicAdd(a.stat_cum, static_cast<unsigned long long>(cum));
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

uint32_t traverse_launch_count(const TraverseArgs& a) {
    const char tv = a.mode;
    return a.nq != 0 && a.k_half <= 128 && rank_rec_fits(a.k_half, a.K) && (tv == 0 || tv == 'r') ? 2u : 1u;
}

cudaError_t launch_traverse(const TraverseArgs& a, cudaStream_t st) {
    if (a.nq == 0) return cudaSuccess;
    const char tv = a.mode;  // Tuning::traverse (tests): 'w' forces the warp-per-task kernel
    const bool warp_path = tv == 'w';
    if (a.k_half <= 128 && !warp_path) {
        const uint32_t L = a.k_half <= 64 ? 64 : 128;
        // two-phase (default): warp-per-half ranking at full occupancy, then the thread-per-task merge
        // ('r' forces it, 't' / 's' / 'n' force the one-kernel thread path)
        const bool two_phase = rank_rec_fits(a.k_half, a.K) && (tv == 0 || tv == 'r');
        if (two_phase) {
            const size_t per_t = size_t(L) * 9 + size_t(a.k_half) * 19;
            // most resident tasks per SM, the cell sizes staged in shared memory or left in global
            size_t fixed = 16;
            uint32_t best_T = 0, best_res = 0;
            bool cs_global = false;
            for (int g = 0; g < 2; ++g) {
                const size_t fx = g ? 16 : size_t(a.K) * 4 + 16;
                for (uint32_t T = 32; T <= 256; T += 32) {
                    const size_t smem = fx + per_t * T;
                    if (smem > 227 * 1024) break;
                    const uint32_t res = static_cast<uint32_t>((228 * 1024) / (smem + 1024)) * T;
                    if (res > best_res || (g && res == best_res && T == best_T)) {
                        best_res = res;
                        best_T = T;
                        fixed = fx;
                        cs_global = g != 0;
                    }
                }
            }
            if (best_T) {
                const uint32_t U = (a.k_half + 31) / 32;
                auto rk = U == 1 ? rank_halves_kernel<1> : U == 2 ? rank_halves_kernel<2> : U == 3 ? rank_halves_kernel<3>
                                                                                                   : rank_halves_kernel<4>;
                const size_t rsmem = kRankWarps * (size_t(a.k_half) * 8 + size_t(a.hmax) * 4 + 128);
                cudaError_t e = cudaSuccess;
                if (rsmem > 48 * 1024) {
                    e = cudaFuncSetAttribute(rk, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(rsmem));
                    if (e != cudaSuccess) return e;
                }
                rk<<<dim3(static_cast<unsigned>((a.nq + kRankWarps - 1) / kRankWarps), 2 * a.ns), 32 * kRankWarps, rsmem,
                     st>>>(a);
                e = cudaGetLastError();
                if (e != cudaSuccess) return e;
                const size_t smem = fixed + per_t * best_T;
                auto kern = L == 64 ? traverse_thread_kernel<64, 1, true> : traverse_thread_kernel<128, 1, true>;
                e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
                if (e != cudaSuccess) return e;
                TraverseArgs b = a;
                b.cs_global = cs_global ? 1u : 0u;
                kern<<<dim3(static_cast<unsigned>((a.nq + best_T - 1) / best_T), a.ns), best_T, smem, st>>>(b);
                return cudaGetLastError();
            }
        }
        // two threads per task measured faster with short halves and small tables (cfg1/cfg2:
        // 0.64 -> 0.60 ms) and slower otherwise (cfg3, h = 30: 0.25 -> 0.34 ms; cfg4, K = 4096:
        // 1.13 -> 1.17 ms); Tuning::traverse 's' / 'n' force it
        const bool split = tv == 's' ? true : tv == 'n' ? false : (a.K <= 2500 && a.hmax <= 16);
        const uint32_t sp = split ? 2u : 1u;  // threads per task (4 measured slower)
        // per task: tkey (L f64), d1r/d2r (2k f64), qh (hmax f32), trow (L), o1/o2/cur (3k u8);
        // split: + the second half's scratch (k f64) and projected query (hmax f32)
        const size_t per_t = size_t(L) * 9 + size_t(a.k_half) * (split ? 27 : 19) + size_t(a.hmax) * (split ? 8 : 4);
        const size_t fixed = size_t(a.K) * 4 + 16;
        uint32_t best_T = 0, best_res = 0;
        for (uint32_t T = 32; T <= 256 && T * sp <= 1024; T += 32) {  // most resident tasks per SM within 227 KB / CTA
            const size_t smem = fixed + per_t * T;
            if (smem > 227 * 1024) break;
            const uint32_t res = static_cast<uint32_t>((228 * 1024) / (smem + 1024)) * T;
            if (res > best_res) {
                best_res = res;
                best_T = T;
            }
        }
        if (best_T) {  // measured faster at every bench config (cfg1 0.22 -> 0.19 ms, cfg2 1.25 -> 0.64)
            const size_t smem = fixed + per_t * best_T;
            auto kern = sp == 2 ? (L == 64 ? traverse_thread_kernel<64, 2> : traverse_thread_kernel<128, 2>)
                                : (L == 64 ? traverse_thread_kernel<64, 1> : traverse_thread_kernel<128, 1>);
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
            if (e != cudaSuccess) return e;
            const dim3 grid(static_cast<unsigned>((a.nq + best_T - 1) / best_T), a.ns);
            kern<<<grid, best_T * sp, smem, st>>>(a);
            return cudaGetLastError();
        }
    }
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
