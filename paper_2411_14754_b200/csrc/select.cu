// Stage 2 of the query path: SC-score counting and top-m candidate selection.
//
// Reference semantics (query.cpp:210-260): every point in every retrieved
// cell of every subspace gets one collision; the candidate set is the top
// m = candidate_count(beta, n, k) points by (score desc, id asc) over all n
// (points never retrieved score 0, so the `touched < m` branch is the T = 0
// case below).
//
// B200 design. One thread-block cluster of CS CTAs owns one query. CTA r
// owns the id slabs r, r + CS, r + 2CS, ... (slab j = ids [j*CH, (j+1)*CH)),
// and keeps that slab's collision counters as u8 in shared memory — scores
// are <= N_s <= 255, so 1 byte per point; counters never touch HBM.
//   * count:  per subspace, the retrieved cells' sub-slices inside the slab
//             (precomputed slab offsets; the IMI keeps ids ascending per cell,
//             index.cpp:90-94) are flattened over the CTA's 16 warps; each
//             lane streams ids (coalesced) and bumps its counter with a plain
//             byte RMW. Within one subspace every id occurs once, so the only
//             ordering needed is a barrier between subspaces.
//   * histogram: SWAR popcounts give, per slab, #points with score >= t for
//             every t.
//   * select: the cluster exchanges slab histograms over DSMEM; every CTA
//             derives the same threshold T (largest t with #(score >= t) >= m)
//             and, walking slabs in id order, the tie quota of each slab —
//             the first `need` points with score == T in id order are taken,
//             which is exactly the reference's (score desc, id asc) cut.
//   * emit:   warp-ordered prefix sums place each selected id at its final
//             position, so the candidate list comes out sorted by id.
// When n > CS * CH_MAX the cluster walks `rounds` slabs per CTA twice
// (histogram pass, then recount + emit) instead of spilling counters.
#include <algorithm>
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace suco_gpu {
namespace {

#ifndef SUCO_SELECT_THREADS
#define SUCO_SELECT_THREADS 1024  // 32 warps/SM: measured best with 4-unit waves (18.7 ms vs 21.4 ms at 512 x 8)
#endif
constexpr uint32_t kThreads = SUCO_SELECT_THREADS;
#ifndef SUCO_SELECT_MINB
#define SUCO_SELECT_MINB 1
#endif
constexpr uint32_t kWarps = kThreads / 32;
constexpr uint32_t kCap = 4 * kThreads;  // retrieved cells staged per chunk (4 per thread)
#ifndef SUCO_SELECT_UNITS
#define SUCO_SELECT_UNITS 4096
#endif
constexpr uint32_t kUnits = 8 * kThreads < SUCO_SELECT_UNITS ? 8 * kThreads : SUCO_SELECT_UNITS;  // 32-id units per window
constexpr uint32_t kFull = 0xffffffffu;
constexpr uint32_t kChAlign = 4 * 32 * kWarps;  // CH multiple of this: whole words per lane-step
constexpr uint32_t kSmemLimit = 232448;        // opt-in dynamic shared memory per block on sm_100

__host__ __device__ inline uint32_t hist_stride(uint32_t ns) { return ns + 2; }

// Cluster-wide barrier with release/acquire at cluster scope (what DSMEM
// visibility needs); cg::cluster_group::sync() additionally fences at GPU scope.
__device__ __forceinline__ void cluster_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

struct Smem {
    uint8_t* cnt;        // CH
    uint32_t* hist;      // rounds x hist_stride: [0] = slab length, [t] = #score >= t
    uint2* udesc;        // kUnits: (id position, id count 1..32) of each 32-id unit
    uint32_t* wtmp;      // 2 * kWarps
    uint32_t* rquota;    // rounds
    uint32_t* roff;      // rounds
    uint32_t* misc;      // 8
    uint32_t* sub_start; // ns + 1: first staged cell of each subspace
    uint32_t* sub_unit;  // ns + 1: first unit of each subspace (chunk-relative)
    uint32_t* hscratch;  // ns + 2: histogram sink of the recount pass
};

__host__ __device__ inline size_t smem_bytes(uint32_t CH, uint32_t rounds, uint32_t ns) {
    return CH + 8ull * kUnits + 4ull * (rounds * hist_stride(ns) + 2 * kWarps + 2 * rounds + 8 + 3 * 257) + 16;
}

__device__ inline Smem carve(unsigned char* base, uint32_t CH, uint32_t rounds, uint32_t ns) {
    Smem s;
    s.cnt = base;
    s.udesc = reinterpret_cast<uint2*>(base + CH);
    s.hist = reinterpret_cast<uint32_t*>(s.udesc + kUnits);
    s.wtmp = s.hist + rounds * hist_stride(ns);
    s.rquota = s.wtmp + 2 * kWarps;
    s.roff = s.rquota + rounds;
    s.misc = s.roff + rounds;
    s.sub_start = s.misc + 8;
    s.sub_unit = s.sub_start + 257;
    s.hscratch = s.sub_unit + 257;
    return s;
}

// Block-wide exclusive scan of one u32 per thread; returns the prefix, total in *tot.
__device__ inline uint32_t block_excl_scan(uint32_t v, uint32_t* wtmp, uint32_t* tot) {
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, off);
        if (lane >= (uint32_t)off) x += y;
    }
    if (lane == 31) wtmp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < kWarps ? wtmp[lane] : 0;
        uint32_t inc = w;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, inc, off);
            if (lane >= (uint32_t)off) inc += y;
        }
        if (lane < kWarps) wtmp[kWarps + lane] = inc - w;
        if (lane == kWarps - 1) wtmp[0] = inc;  // total (wtmp[0] already consumed above)
    }
    __syncthreads();
    const uint32_t res = wtmp[kWarps + warp] + (x - v);
    *tot = wtmp[0];
    __syncthreads();
    return res;
}

// ---------------------------------------------------------------- counting
// Per-thread histogram of the values produced by increments, 8-bit fields
// (bin v-1 in byte (v-1)&7 of word (v-1)>>3). An id with final score s is
// incremented through 1..s, so #increments producing v == #ids with score >= v.
// A lane adds at most 16 per wave, so flushing every 15 waves cannot overflow.
template <int NSB>
struct IncHist {
    static constexpr int W = NSB > 0 ? (NSB + 7) / 8 : 1;
    uint64_t h[W];
    __device__ void clear() {
#pragma unroll
        for (int i = 0; i < W; ++i) h[i] = 0;
    }
    __device__ __forceinline__ void add(uint32_t v, uint32_t* hist_smem) {
        if constexpr (NSB > 0) {
            const uint32_t b = v - 1;
            if constexpr (W == 1) {
                h[0] += 1ull << (8u * b);
            } else {
                const uint64_t inc = 1ull << (8u * (b & 7u));
#pragma unroll
                for (int i = 0; i < W; ++i) h[i] += ((b >> 3) == (uint32_t)i) ? inc : 0ull;
            }
        } else {
            atomicAdd(hist_smem + v, 1u);
        }
    }
    // warp-reduce and add into hist[1..ns]; clears the fields
    __device__ void flush(uint32_t* hist, uint32_t ns) {
        if constexpr (NSB > 0) {
            const uint32_t lane = threadIdx.x & 31u;
#pragma unroll
            for (int b = 0; b < NSB; ++b) {
                uint32_t v = static_cast<uint32_t>((h[b >> 3] >> ((b & 7) * 8)) & 0xffu);
                if (__any_sync(kFull, v != 0)) {
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
                    if (lane == 0 && (uint32_t)b < ns) atomicAdd(hist + b + 1, v);
                }
            }
            clear();
        }
    }
};

template <int KU>
struct Wave {
    uint32_t id[KU];
    uint32_t mask;  // bit u: entry u valid for this lane
};

// Loads wave [ua, ub) of 32-id units (at most KU units): lane l takes id l of
// each unit; every slot is predicated (invalid slots re-read unit ua and issue no
// global load). Used by the generic (N_s > 32) counting loop.
template <int KU>
__device__ __forceinline__ void load_wave(const Smem& s, const uint32_t* ids, uint32_t ua, uint32_t ub, Wave<KU>& w) {
    const uint32_t lane = threadIdx.x & 31u;
    uint32_t mask = 0;
#pragma unroll
    for (int u = 0; u < KU; ++u) {
        const uint32_t unit = ua + u < ub ? ua + u : ua;
        const uint2 d = s.udesc[unit];  // (begin, count)
        const bool ok = (ua + u < ub) && (lane < d.y);
        w.id[u] = ok ? __ldg(ids + d.x + lane) : 0u;
        mask |= static_cast<uint32_t>(ok) << u;
    }
    w.mask = mask;
}

// ---- lean (branch-free) waves. Shared memory is addressed with 32-bit
// shared-window addresses computed once (plain pointers made the compiler
// rebuild the cluster window base, S2R SR_CgaCtaId + LEA, on every access), one
// LDS.64 per unit descriptor, a predicated global load per slot, and invalid
// slots redirected to a scratch byte with produced value 0 (whose histogram
// increment is shl(1, 0xfffffff8) = 0 under PTX's clamped shifts).
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint2 lds_v2(uint32_t a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_u8(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v));
}
// Predicated load; the result is undefined when !ok (callers mask it).
__device__ __forceinline__ uint32_t ldg_if(const uint32_t* p, bool ok) {
    uint32_t v = 0;
    asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.global.nc.u32 %0, [%1];\n\t}"
        : "+r"(v)
        : "l"(p), "r"(static_cast<uint32_t>(ok)));
    return v;
}
// Opaque copy: keeps a loop invariant in a register (otherwise the compiler
// rematerializes shared-window addresses from SR_CgaCtaId inside the loop).
__device__ __forceinline__ uint32_t pin(uint32_t x) {
    uint32_t y;
    asm volatile("mov.b32 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}
__device__ __forceinline__ uint64_t one_shl(uint32_t sh) {  // 1 << sh, 0 when sh >= 64
    uint64_t r;
    asm("shl.b64 %0, %1, %2;" : "=l"(r) : "l"(1ull), "r"(sh));
    return r;
}

template <int NSB>
__device__ __forceinline__ void hist_add_lean(IncHist<NSB>& ih, uint32_t v) {  // v = 0: no-op
    const uint32_t b = v - 1u;
    if constexpr (IncHist<NSB>::W == 1) {
        ih.h[0] += one_shl(8u * b);
    } else {
        const uint64_t inc = one_shl(8u * (b & 7u));
#pragma unroll
        for (int i = 0; i < IncHist<NSB>::W; ++i) ih.h[i] += ((b >> 3) == (uint32_t)i) ? inc : 0ull;
    }
}

template <int KU>
__device__ __forceinline__ void load_wave_lean(uint32_t ud_sa, const uint32_t* ids, uint32_t ua, uint32_t ub,
                                               uint32_t lane, Wave<KU>& w) {
    uint32_t mask = 0;
#pragma unroll
    for (int u = 0; u < KU; ++u) {
        const bool in = ua + u < ub;  // warp-uniform; past-the-end descriptors read in-bounds junk, masked below
        const uint2 d = lds_v2(ud_sa + 8u * (ua + u));
        const bool ok = in && lane < d.y;
        w.id[u] = ldg_if(ids + (d.x + lane), ok);
        mask |= static_cast<uint32_t>(ok) << u;
    }
    w.mask = mask;
}

// cbase = shared address of counter 0 minus the slab's first id (wraps mod 2^32).
template <int NSB, int KU>
__device__ __forceinline__ void rmw_wave_lean(uint32_t cbase, uint32_t dummy, const Wave<KU>& w, IncHist<NSB>& ih) {
    uint32_t ad[KU], v[KU];
#pragma unroll
    for (int u = 0; u < KU; ++u) ad[u] = ((w.mask >> u) & 1u) ? cbase + w.id[u] : dummy;
#pragma unroll
    for (int u = 0; u < KU; ++u) v[u] = lds_u8(ad[u]);
#pragma unroll
    for (int u = 0; u < KU; ++u) v[u] = ((w.mask >> u) & 1u) ? v[u] + 1u : 0u;
#pragma unroll
    for (int u = 0; u < KU; ++u) sts_u8(ad[u], v[u]);
#pragma unroll
    for (int u = 0; u < KU; ++u) hist_add_lean<NSB>(ih, v[u]);
}

template <int NSB, int KU>
__device__ __forceinline__ void rmw_wave(const Smem& s, const Wave<KU>& w, uint32_t lo, IncHist<NSB>& ih,
                                         uint32_t* hist) {
    // Every slot of a wave holds a different id (one subspace, distinct units /
    // lanes), so all counter reads can be issued before any write.
    uint32_t v[KU];
#pragma unroll
    for (int u = 0; u < KU; ++u) v[u] = (w.mask & (1u << u)) ? s.cnt[w.id[u] - lo] + 1u : 0u;
#pragma unroll
    for (int u = 0; u < KU; ++u) {
        if (w.mask & (1u << u)) {
            s.cnt[w.id[u] - lo] = static_cast<uint8_t>(v[u]);
            ih.add(v[u], hist);
        }
    }
}

// Counts one slab into s.cnt (query.cpp:235-239 restricted to the slab) and
// fills hist[t] = #counters >= t (t = 1..ns), hist[0] = len.
//
// Staging: each thread loads the slab slice (begin, length) of 4 retrieved
// cells (all subspaces at once), a block scan over ceil(length/32) cuts every
// slice into 32-id "units", and the unit descriptors (begin, count) go to
// shared memory. Counting: each subspace's units are split evenly over the
// 16 warps; a warp loads kU units (one id per lane per unit, coalesced) and
// then does the counter RMWs, with the first wave of subspace s+1 already in
// flight while subspace s does its RMWs. A barrier separates subspaces (an id
// repeats only across subspaces).
template <int NSB, int KU>
__device__ void count_slab(const SelectArgs& a, const Smem& s, uint64_t q, uint32_t slab, uint64_t lo, uint32_t len,
                           uint32_t* hist) {
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    uint4* c4 = reinterpret_cast<uint4*>(s.cnt);
    for (uint32_t i = tid; i < a.CH / 16; i += kThreads) c4[i] = make_uint4(0, 0, 0, 0);
    if (tid <= a.ns) hist[tid] = tid == 0 ? len : 0u;
    if (tid == 0) {
        uint32_t acc = 0;
        for (uint32_t sub = 0; sub < a.ns; ++sub) {
            s.sub_start[sub] = acc;
            acc += a.ncells[q * a.ns + sub];
        }
        s.sub_start[a.ns] = acc;
    }
    __syncthreads();
    if (len == 0) return;
    const uint32_t TC = s.sub_start[a.ns];
    const uint32_t stride = a.nslabs + 1;
    // lean waves address ids by one 32-bit offset into the N_s x n array when it fits
    const bool abs_ids = NSB > 0 && static_cast<uint64_t>(a.ns) * a.n <= 0xffffffffull;
    IncHist<NSB> ih;
    ih.clear();
    uint32_t waves_since_flush = 0;
    for (uint32_t c0 = 0; c0 < TC; c0 += kCap) {
        const uint32_t c1 = min(TC, c0 + kCap);
        // stage 4 consecutive cells per thread: (begin, length) -> units
        uint32_t beg4[4] = {0, 0, 0, 0}, len4[4] = {0, 0, 0, 0}, nu4[4] = {0, 0, 0, 0};
        const uint32_t g0 = c0 + 4 * tid;
        uint32_t sub = 0;
        while (sub + 1 < a.ns && s.sub_start[sub + 1] <= g0) ++sub;
        const uint32_t sub_first = sub;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t g = g0 + u;
            if (g < c1) {
                while (s.sub_start[sub + 1] <= g) ++sub;
                const uint32_t cell = __ldg(a.cells + (q * a.ns + sub) * a.cells_cap + (g - s.sub_start[sub]));
                const uint32_t* p = a.slab_off + (static_cast<uint64_t>(sub) * a.K + cell) * stride + slab;
                beg4[u] = __ldg(p);
                len4[u] = __ldg(p + 1) - beg4[u];
                nu4[u] = (len4[u] + 31) >> 5;
                if (abs_ids) beg4[u] += sub * static_cast<uint32_t>(a.n);  // offset into the whole N_s x n array
            }
        }
        uint32_t UT;
        const uint32_t up0 = block_excl_scan(nu4[0] + nu4[1] + nu4[2] + nu4[3], s.wtmp, &UT);
        // unit index where each subspace starts within this chunk
        {
            uint32_t up = up0, sb2 = sub_first;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t g = g0 + u;
                if (g < c1) {
                    while (s.sub_start[sb2 + 1] <= g) ++sb2;
                    if (g == s.sub_start[sb2] || g == c0) s.sub_unit[sb2] = up;
                }
                up += nu4[u];
            }
            if (tid == 0) {
                // subspaces that start at or before c0 begin at unit 0; those past c1 at UT
                for (uint32_t t = 0; t <= a.ns; ++t) {
                    if (s.sub_start[t] >= c1) s.sub_unit[t] = UT;
                }
            }
        }
        __syncthreads();
        uint32_t sb = 0;
        while (sb + 1 < a.ns && s.sub_start[sb + 1] <= c0) ++sb;
        uint32_t se = sb;
        while (se < a.ns && s.sub_start[se] < c1) ++se;  // subspaces [sb, se) overlap the chunk

        for (uint32_t u0 = 0; u0 < UT; u0 += kUnits) {
            const uint32_t u1 = min(UT, u0 + kUnits);
            // describe the units of this window
            {
                uint32_t up = up0;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    for (uint32_t j = 0; j < nu4[u]; ++j) {
                        const uint32_t unit = up + j;
                        if (unit >= u0 && unit < u1) {
                            s.udesc[unit - u0] = make_uint2(beg4[u] + 32u * j, min(32u, len4[u] - 32u * j));
                        }
                    }
                    up += nu4[u];
                }
            }
            __syncthreads();
            auto range = [&](uint32_t sb3, uint32_t& ua, uint32_t& ub) {
                const uint32_t A = max(s.sub_unit[sb3], u0) - u0;
                const uint32_t B = max(min(s.sub_unit[sb3 + 1], u1), u0) - u0;
                const uint32_t T = B > A ? B - A : 0;
                ua = A + static_cast<uint32_t>((static_cast<uint64_t>(T) * warp) / kWarps);
                ub = A + static_cast<uint32_t>((static_cast<uint64_t>(T) * (warp + 1)) / kWarps);
            };
            if constexpr (NSB > 0) {
                // lean waves (a wave is loaded then RMW'd; one barrier per subspace). Measured
                // slower: carrying the next subspace's first wave over the barrier (register
                // pressure) and an mbarrier split arrive/wait (1024 threads polling).
                const uint32_t ud_sa = smem_addr(s.udesc);
                const uint32_t cbase = pin(smem_addr(s.cnt) - static_cast<uint32_t>(lo));
                const uint32_t dummy = smem_addr(s.misc + 7);
                for (uint32_t sb3 = sb; sb3 < se; ++sb3) {
                    uint32_t ua, ub;
                    range(sb3, ua, ub);
                    const uint32_t* ids = abs_ids ? a.ids : a.ids + static_cast<uint64_t>(sb3) * a.n;
                    for (uint32_t u0 = ua; u0 < ub; u0 += KU) {
                        Wave<KU> w;
                        load_wave_lean<KU>(ud_sa, ids, u0, ub, lane, w);
                        __syncwarp();  // keeps ptxas from hoisting a slot's RMW above the other slots' loads
                        rmw_wave_lean<NSB, KU>(cbase, dummy, w, ih);
                        if (++waves_since_flush * KU >= 240) {
                            ih.flush(hist, a.ns);
                            waves_since_flush = 0;
                        }
                    }
                    __syncthreads();  // counters of sb3 final before sb3 + 1 increments
                }
            } else {
                for (uint32_t sb3 = sb; sb3 < se; ++sb3) {
                    uint32_t ua, ub;
                    range(sb3, ua, ub);
                    const uint32_t* ids = a.ids + static_cast<uint64_t>(sb3) * a.n;
                    for (uint32_t u0 = ua; u0 < ub; u0 += KU) {
                        Wave<KU> w;
                        load_wave<KU>(s, ids, u0, ub, w);
                        rmw_wave<NSB, KU>(s, w, static_cast<uint32_t>(lo), ih, hist);
                        if (++waves_since_flush * KU >= 240) {
                            ih.flush(hist, a.ns);
                            waves_since_flush = 0;
                        }
                    }
                    __syncthreads();  // counters of sb3 final before sb3 + 1 increments
                }
            }
        }
    }
    ih.flush(hist, a.ns);
    __syncthreads();
}

// Mask (0x80 per byte) of the bytes of word `wi` that are >= t and inside the slab.
__device__ __forceinline__ uint32_t sel_mask(uint32_t w, uint32_t wi, uint32_t t, uint32_t len, bool swar) {
    uint32_t m;
    if (t == 0) {
        m = 0x80808080u;
    } else if (swar) {
        m = (w + (0x80u - t) * 0x01010101u) & 0x80808080u;
    } else {
        m = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) m |= (((w >> (8 * b)) & 0xffu) >= t) ? (0x80u << (8 * b)) : 0u;
    }
    const uint32_t valid = wi * 4 + 4 <= len ? 4u : (len > wi * 4 ? len - wi * 4 : 0u);
    if (valid < 4) m &= (1u << (8 * valid)) - 1u;
    return m;
}

// Emits this slab's share of the candidate set into cands[base, base + gt + quota):
// every counter > T (and, when the slab's whole tie class is taken, every
// counter == T) goes out unordered through a warp-aggregated shared counter —
// the candidate SET is what the reference defines (query.cpp:242-260); only
// the slab where the tie quota is cut needs id order, and only for its ties,
// which a two-pass warp-ordered scan emits after the unordered region.
__device__ void emit_slab(const SelectArgs& a, const Smem& s, uint64_t q, uint64_t lo, uint32_t len, uint32_t T,
                          uint32_t quota, uint32_t base, uint32_t gt, uint32_t ties, bool swar) {
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint4* w128 = reinterpret_cast<const uint4*>(s.cnt);
    const uint32_t words = (len + 3) / 4;
    const uint32_t nvec = (words + 3) / 4;
    uint32_t* out = a.cands + q * a.m + base;
    const bool all_ties = quota == ties;
    const uint32_t tsel = all_ties ? T : T + 1;
    if (tid == 0) s.misc[1] = 0;
    __syncthreads();
    if (gt + (all_ties ? ties : 0u) > 0) {
        // vectors [0, full) lie inside the slab; at most one partial vector follows.
        // One flag word per 16-counter vector: the four 0x80-per-byte masks folded as
        // m0 | m1 >> 1 | m2 >> 2 | m3 >> 3, so bit p <-> counter (7 - p % 8) * 4 + p / 8
        // and a single POPC counts the vector (POPC is quarter rate).
        const uint32_t full = len / 16;
        const uint32_t kq = (0x80u - (tsel ? tsel : 1u)) * 0x01010101u;
        const uint32_t w_sa = smem_addr(s.cnt);
        auto flags = [&](uint32_t vi) -> uint32_t {
            uint4 v;
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                         : "r"(w_sa + 16u * vi));
            uint32_t m0, m1, m2, m3;
            if (tsel == 0) {
                m0 = m1 = m2 = m3 = 0x80808080u;
            } else if (swar) {
                m0 = (v.x + kq) & 0x80808080u;
                m1 = (v.y + kq) & 0x80808080u;
                m2 = (v.z + kq) & 0x80808080u;
                m3 = (v.w + kq) & 0x80808080u;
            } else {
                m0 = sel_mask(v.x, 0, tsel, 4, false);
                m1 = sel_mask(v.y, 0, tsel, 4, false);
                m2 = sel_mask(v.z, 0, tsel, 4, false);
                m3 = sel_mask(v.w, 0, tsel, 4, false);
            }
            if (vi >= full) {  // the partial tail vector
                m0 &= sel_mask(0xffffffffu, vi * 4 + 0, 0, len, true);
                m1 &= sel_mask(0xffffffffu, vi * 4 + 1, 0, len, true);
                m2 &= sel_mask(0xffffffffu, vi * 4 + 2, 0, len, true);
                m3 &= sel_mask(0xffffffffu, vi * 4 + 3, 0, len, true);
            }
            return m0 | (m1 >> 1) | (m2 >> 2) | (m3 >> 3);
        };
        constexpr uint32_t kV = 4;  // vectors per lane per step (64 counters)
        for (uint32_t v0 = 0; v0 < nvec; v0 += kThreads * kV) {
            uint32_t f[kV];
            uint32_t c = 0;
#pragma unroll
            for (uint32_t j = 0; j < kV; ++j) {
                const uint32_t vi = v0 + j * kThreads + tid;
                f[j] = vi < nvec ? flags(vi) : 0u;
                c += __popc(f[j]);
            }
            if (!__any_sync(kFull, c != 0)) continue;
            uint32_t x = c;  // warp-aggregated slot reservation (emission order is free)
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t y = __shfl_up_sync(kFull, x, off);
                if (lane >= (uint32_t)off) x += y;
            }
            uint32_t wbase = 0;
            if (lane == 31) wbase = atomicAdd(&s.misc[1], x);
            wbase = __shfl_sync(kFull, wbase, 31);
            uint32_t pos = wbase + x - c;
#pragma unroll
            for (uint32_t j = 0; j < kV; ++j) {
                uint32_t mm = f[j];
                const uint32_t idb = static_cast<uint32_t>(lo) + (v0 + j * kThreads + tid) * 16u;
                while (mm) {
                    const uint32_t p = __ffs(mm) - 1;
                    __stcs(out + pos++, idb + (7u - (p & 7u)) * 4u + (p >> 3));  // streaming: keep ids in L2
                    mm &= mm - 1;
                }
            }
        }
    }
    if (all_ties || quota == 0) return;
    // boundary slab: the first `quota` ties (== T) in id order, after the gt
    // region. Warps own contiguous vector ranges; lanes step over 16-counter
    // vectors, so both passes read shared memory conflict-free.
    uint32_t* tout = out + gt;
    const uint32_t last_vi = (len - 1) / 16;
    const uint32_t kT = (0x80u - (T ? T : 1u)) * 0x01010101u, kT1 = (0x80u - (T + 1)) * 0x01010101u;
    auto tie_mask = [&](uint32_t w) -> uint32_t {
        if (!swar) return sel_mask(w, 0, T, 4, false) & ~sel_mask(w, 0, T + 1, 4, false);
        const uint32_t ge1 = (w + kT1) & 0x80808080u;
        const uint32_t ge0 = T ? ((w + kT) & 0x80808080u) : 0x80808080u;
        return ge0 & ~ge1;
    };
    auto vec_ties = [&](uint32_t vi, uint32_t (&mt)[4]) {
        const uint4 v = w128[vi];
        mt[0] = tie_mask(v.x);
        mt[1] = tie_mask(v.y);
        mt[2] = tie_mask(v.z);
        mt[3] = tie_mask(v.w);
        if (vi == last_vi) {
#pragma unroll
            for (int u = 0; u < 4; ++u) mt[u] &= sel_mask(0xffffffffu, vi * 4 + u, 0, len, true);
        }
    };
    const uint32_t vpw = (nvec + kWarps - 1) / kWarps;
    const uint32_t va = min(nvec, warp * vpw), vb = min(nvec, va + vpw);
    uint32_t e_tot = 0;
    for (uint32_t vi = va + lane; vi < vb; vi += 32) {
        uint32_t mt[4];
        vec_ties(vi, mt);
        e_tot += __popc(mt[0]) + __popc(mt[1]) + __popc(mt[2]) + __popc(mt[3]);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) e_tot += __shfl_xor_sync(kFull, e_tot, off);
    uint32_t tmp;
    const uint32_t e_base = block_excl_scan(lane == 0 ? e_tot : 0u, s.wtmp, &tmp);
    uint32_t eb = __shfl_sync(kFull, e_base, 0);
    for (uint32_t v0 = va; v0 < vb && eb < quota; v0 += 32) {
        const uint32_t vi = v0 + lane;
        uint32_t mt[4] = {0, 0, 0, 0};
        if (vi < vb) vec_ties(vi, mt);
        const uint32_t e = __popc(mt[0]) + __popc(mt[1]) + __popc(mt[2]) + __popc(mt[3]);
        uint32_t ex = e;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, ex, off);
            if (lane >= (uint32_t)off) ex += y;
        }
        const uint32_t esum = __shfl_sync(kFull, ex, 31);
        uint32_t r = eb + ex - e;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            uint32_t mm = mt[u];
            while (mm && r < quota) {
                const uint32_t bit = __ffs(mm) - 1;
                __stcs(tout + r++, static_cast<uint32_t>(lo) + (vi * 4 + u) * 4 + (bit >> 3));
                mm &= mm - 1;
            }
        }
        eb += esum;
    }
}

template <int NSB, int KU = 4>
__global__ void __launch_bounds__(kThreads, SUCO_SELECT_MINB) select_kernel(SelectArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    cg::cluster_group cluster = cg::this_cluster();
    const uint32_t rank = cluster.block_rank();
    const Smem s = carve(smem, a.CH, a.rounds, a.ns);
    const uint32_t hs = hist_stride(a.ns);
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const bool swar = a.ns <= 127;
    // persistent clusters: cluster c handles queries c, c + C, c + 2C, ...
    const uint64_t nclusters = gridDim.x / a.CS;
    for (uint64_t q = blockIdx.x / a.CS; q < a.nq; q += nclusters) {

        // pass 1: count + histogram every owned slab
        for (uint32_t r = 0; r < a.rounds; ++r) {
            const uint32_t slab = r * a.CS + rank;
            const uint64_t lo = static_cast<uint64_t>(slab) * a.CH;
            const uint32_t len = slab < a.nslabs ? static_cast<uint32_t>(min_u64(a.CH, a.n - lo)) : 0u;
            count_slab<NSB, KU>(a, s, q, slab, lo, len, s.hist + r * hs);
            if (a.scores_dbg) {
                const uint64_t ss = a.scores_stride ? a.scores_stride : a.n;
                uint8_t* dst = a.scores_dbg + q * ss + lo;
                if ((ss & 15u) == 0) {  // 16-byte rows: vector copy (lo is a multiple of CH)
                    const uint32_t nv = len / 16;
                    for (uint32_t i = tid; i < nv; i += kThreads) {
                        reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(s.cnt)[i];
                    }
                    for (uint32_t i = nv * 16 + tid; i < len; i += kThreads) dst[i] = s.cnt[i];
                } else {
                    for (uint32_t i = tid; i < len; i += kThreads) dst[i] = s.cnt[i];
                }
            }

        }
        cluster_barrier();

        // threshold and per-slab quotas (warp 0), from every slab's histogram
        if (warp == 0) {
            const uint32_t G = a.nslabs;
            uint32_t tot[NSB > 0 ? NSB + 1 : 1];
            uint32_t T = 0;
            uint64_t need = 0;
            if constexpr (NSB > 0) {
    #pragma unroll
                for (int t = 0; t <= NSB; ++t) tot[t] = 0;
                for (uint32_t g = lane; g < G; g += 32) {
                    const uint32_t* h = cluster.map_shared_rank(s.hist, g % a.CS) + (g / a.CS) * hs;
    #pragma unroll
                    for (int t = 1; t <= NSB; ++t) {
                        if ((uint32_t)t <= a.ns) tot[t] += h[t];
                    }
                }
    #pragma unroll
                for (int t = 1; t <= NSB; ++t) {
    #pragma unroll
                    for (int off = 16; off > 0; off >>= 1) tot[t] += __shfl_xor_sync(kFull, tot[t], off);
                }
                for (int t = NSB; t >= 1; --t) {
                    if ((uint32_t)t <= a.ns && tot[t] >= a.m) {
                        T = t;
                        break;
                    }
                }
                uint32_t gt_total = 0;
    #pragma unroll
                for (int t = 1; t <= NSB; ++t) {
                    if ((uint32_t)t == T + 1 && (uint32_t)t <= a.ns) gt_total = tot[t];
                }
                need = a.m - gt_total;
            } else {
                // generic (N_s > 32): one level at a time, top down
                uint64_t prev = 0;
                T = 0;
                need = a.m;
                for (uint32_t t = a.ns; t >= 1; --t) {
                    uint32_t c = 0;
                    for (uint32_t g = lane; g < G; g += 32) {
                        c += (cluster.map_shared_rank(s.hist, g % a.CS) + (g / a.CS) * hs)[t];
                    }
    #pragma unroll
                    for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(kFull, c, off);
                    if (c >= a.m) {
                        T = t;
                        need = a.m - prev;
                        break;
                    }
                    prev = c;
                }
                if (T == 0) need = a.m - prev;
            }
            // quotas in global slab (= id) order
            uint64_t ties_run = 0, out_run = 0;
            for (uint32_t g0 = 0; g0 < G; g0 += 32) {
                const uint32_t g = g0 + lane;
                uint32_t ties = 0, gt = 0;
                if (g < G) {
                    const uint32_t* h = cluster.map_shared_rank(s.hist, g % a.CS) + (g / a.CS) * hs;
                    const uint32_t geT = h[T];
                    const uint32_t geT1 = T + 1 <= a.ns ? h[T + 1] : 0u;
                    gt = geT1;
                    ties = geT - geT1;
                }
                uint64_t tx = ties;
    #pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const uint64_t y = __shfl_up_sync(kFull, tx, off);
                    if (lane >= (uint32_t)off) tx += y;
                }
                const uint64_t tsum = __shfl_sync(kFull, tx, 31);
                tx -= ties;
                const uint64_t before = ties_run + tx;
                const uint32_t quota = before >= need ? 0u : static_cast<uint32_t>(min_u64(ties, need - before));
                uint64_t ox = gt + quota;
                const uint64_t mine = ox;
    #pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const uint64_t y = __shfl_up_sync(kFull, ox, off);
                    if (lane >= (uint32_t)off) ox += y;
                }
                const uint64_t osum = __shfl_sync(kFull, ox, 31);
                ox -= mine;
                if (g < G && g % a.CS == rank) {
                    s.rquota[g / a.CS] = quota;
                    s.roff[g / a.CS] = static_cast<uint32_t>(out_run + ox);
                }
                ties_run += tsum;
                out_run += osum;
            }
            if (lane == 0) s.misc[0] = T;
        }
        cluster_barrier();  // peers finished reading our histograms
        const uint32_t T = s.misc[0];

        for (uint32_t r = 0; r < a.rounds; ++r) {
            const uint32_t slab = r * a.CS + rank;
            if (slab >= a.nslabs) break;
            const uint64_t lo = static_cast<uint64_t>(slab) * a.CH;
            const uint32_t len = static_cast<uint32_t>(min_u64(a.CH, a.n - lo));
            if (a.rounds > 1) {
                count_slab<NSB, KU>(a, s, q, slab, lo, len, s.hscratch);  // recount
            }
            const uint32_t* h = s.hist + r * hs;
            const uint32_t gt = T + 1 <= a.ns ? h[T + 1] : 0u;
            emit_slab(a, s, q, lo, len, T, s.rquota[r], s.roff[r], gt, h[T] - gt, swar);
            __syncthreads();
        }
    }
}

__global__ void slab_offsets_kernel(const uint32_t* cell_off, const uint32_t* ids, uint64_t n, uint32_t ns,
                                    uint32_t K, uint32_t CH, uint32_t nslabs, uint32_t* slab_off) {
    const uint64_t stride = nslabs + 1;
    const uint64_t total = static_cast<uint64_t>(ns) * K * stride;
    for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t j = t % stride;
        const uint64_t sc = t / stride;  // s * K + cell
        const uint32_t s = static_cast<uint32_t>(sc / K);
        const uint32_t cell = static_cast<uint32_t>(sc % K);
        const uint32_t* off = cell_off + static_cast<uint64_t>(s) * (K + 1);
        const uint32_t* sid = ids + static_cast<uint64_t>(s) * n;
        uint32_t lo = off[cell], hi = off[cell + 1];
        const uint64_t bound = j * CH;
        while (lo < hi) {  // first position with id >= bound
            const uint32_t mid = lo + ((hi - lo) >> 1);
            if (sid[mid] < bound) lo = mid + 1;
            else hi = mid;
        }
        slab_off[t] = lo;
    }
}

using SelectFn = void (*)(SelectArgs);

template <int NSB>
cudaError_t launch_select_t(const SelectArgs& a, const SelectConfig& cfg, uint64_t nq, cudaStream_t st) {
    const SelectFn fn = select_kernel<NSB>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(cfg.smem));
    if (e != cudaSuccess) return e;
    if (cfg.CS > 8) {
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t lc = {};
    // One cluster per query: measured faster than a persistent grid of resident
    // clusters (the hardware re-fills freed GPC slots dynamically; static
    // round-robin over queries left SMs idle behind the slowest cluster).
    const uint64_t nclusters = nq;
    lc.gridDim = dim3(static_cast<unsigned>(nclusters * cfg.CS));
    lc.blockDim = dim3(kThreads);
    lc.dynamicSmemBytes = cfg.smem;
    lc.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cfg.CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
    return cudaLaunchKernelEx(&lc, fn, a);
}

}  // namespace

cudaError_t launch_select_dispatch(const SelectArgs& a, const SelectConfig& cfg, uint64_t nq, cudaStream_t st);

static SelectConfig plan_for(uint64_t n, uint32_t ns, uint32_t CS) {
    SelectConfig c;
    c.CS = CS;
    c.clusters = 0;
    const uint64_t per = (n + c.CS - 1) / c.CS;
    // largest slab whose counters + unit descriptors + bookkeeping fit the opt-in limit
    uint32_t kChMax = ((kSmemLimit - static_cast<uint32_t>(smem_bytes(0, 1, ns)) - 4096) / kChAlign) * kChAlign;
    {
        const uint64_t slabs = (n + kChMax - 1) / kChMax;
        const uint32_t rounds = static_cast<uint32_t>((slabs + CS - 1) / CS);
        while (kChMax > kChAlign && smem_bytes(kChMax, rounds, ns) > kSmemLimit) kChMax -= kChAlign;
    }
    if (per <= kChMax) {
        c.CH = static_cast<uint32_t>(((per + kChAlign - 1) / kChAlign) * kChAlign);
        if (c.CH == 0) c.CH = kChAlign;
        c.nslabs = static_cast<uint32_t>((n + c.CH - 1) / c.CH);
        c.rounds = 1;
    } else {
        c.CH = kChMax;
        c.nslabs = static_cast<uint32_t>((n + c.CH - 1) / c.CH);
        c.rounds = (c.nslabs + c.CS - 1) / c.CS;
    }
    c.smem = smem_bytes(c.CH, c.rounds, ns);
    return c;
}

template <int NSB>
static int active_clusters(const SelectConfig& c) {
    if (cudaFuncSetAttribute(select_kernel<NSB>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(c.smem)) != cudaSuccess ||
        (c.CS > 8 && cudaFuncSetAttribute(select_kernel<NSB>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)) {
        cudaGetLastError();
        return 0;
    }
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(c.CS * 1024);
    lc.blockDim = dim3(kThreads);
    lc.dynamicSmemBytes = c.smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = c.CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
    int num = 0;
    if (cudaOccupancyMaxActiveClusters(&num, select_kernel<NSB>, &lc) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return num;
}

static int active_clusters_ns(uint32_t ns, const SelectConfig& c) {
    if (ns <= 8) return active_clusters<8>(c);
    if (ns <= 16) return active_clusters<16>(c);
    if (ns <= 32) return active_clusters<32>(c);
    return active_clusters<0>(c);
}


// Cluster size: the one that keeps the most SMs busy with a single counting
// round (clusters must fit inside a GPC, so 8-CTA clusters strand SMs on a
// 148-SM B200); SUCO_CLUSTER (cluster_size > 0) forces a size.
SelectConfig plan_select(uint64_t n, uint32_t ns, int cluster_size) {
    if (cluster_size > 0) {
        SelectConfig c = plan_for(n, ns, static_cast<uint32_t>(cluster_size));
        c.clusters = active_clusters_ns(ns, c);
        return c;
    }
    SelectConfig best = plan_for(n, ns, 8);
    long best_score = -1;
    for (uint32_t cs = 8; cs >= 1; --cs) {
        const SelectConfig c = plan_for(n, ns, cs);
        if (c.rounds > 1 && cs != 8) continue;
        const long score = static_cast<long>(active_clusters_ns(ns, c)) * cs * (c.rounds == 1 ? 2 : 1);
        if (score > best_score) {
            best_score = score;
            best = c;
            best.clusters = static_cast<int>(score / (cs * (c.rounds == 1 ? 2 : 1)));
        }
    }
    return best;
}

cudaError_t launch_select(const SelectArgs& a, const SelectConfig& cfg, uint64_t nq, cudaStream_t st) {
    if (nq == 0) return cudaSuccess;
    return launch_select_dispatch(a, cfg, nq, st);
}

cudaError_t launch_select_dispatch(const SelectArgs& a, const SelectConfig& cfg, uint64_t nq, cudaStream_t st) {
    if (a.ns <= 8) return launch_select_t<8>(a, cfg, nq, st);
    if (a.ns <= 16) return launch_select_t<16>(a, cfg, nq, st);
    if (a.ns <= 32) return launch_select_t<32>(a, cfg, nq, st);
    return launch_select_t<0>(a, cfg, nq, st);
}

cudaError_t launch_slab_offsets(const uint32_t* cell_off, const uint32_t* ids, uint64_t n, uint32_t ns, uint32_t K,
                                uint32_t CH, uint32_t nslabs, uint32_t* slab_off, cudaStream_t st) {
    const uint64_t total = static_cast<uint64_t>(ns) * K * (nslabs + 1);
    const uint64_t blocks = min_u64((total + 255) / 256, 148ull * 16);
    slab_offsets_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(cell_off, ids, n, ns, K, CH, nslabs, slab_off);
    return cudaGetLastError();
}

}  // namespace suco_gpu
