// Dense bit-sliced selection over 32-query blocks (the select stage when
// N_s <= 8 and the per-cell masks fit shared memory).
//
// The SC-score of point p for query q is the number of subspaces s whose
// retrieved cells contain cell_s(p) (query.cpp:229-239: every id of a
// retrieved cell gets one collision, and every id lies in exactly one cell
// per subspace). A CTA owns 32 queries: for every (subspace, cell) it keeps a
// 32-bit mask M[s*K + cell] whose bit j says "query j retrieved this cell".
// A point's 8 masks summed bit-wise by a carry-save adder tree are its 4-bit
// scores for all 32 queries at once (bit-planes b0..b3, bit j = query j); a
// 32x32 bit transpose across the warp turns the planes of 32 consecutive
// points into, per lane = query, the planes of that query's 32 scores. So one
// table lookup serves 32 queries, and every point is visited in id order.
//
// The top-m by (score desc, id asc) (query.cpp:242-260) is cut exactly like
// the shard protocol: points are split into id-contiguous pieces (one per
// warp); K1 writes each piece's #(score >= t), K2 derives per query the
// threshold T, need = m - #(score > T) and each piece's tie quota (the first
// `need` ties in id order) and output offset, K3 re-scores the piece and
// each lane emits its query's candidates: every score > T and the first
// quota ties of the piece in id order.
//
// Point codes: codes[p][s] = s*K + cell_s(p) (u16; s >= N_s -> N_s*K, a
// mask slot that is always zero).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace suco_gpu {
namespace {

// CTA shapes: 512 threads x 2 CTAs/SM when the masks fit 110 KB, else one
// 1024-thread CTA per SM (masks up to 200 KB); a warp = one piece either way.
constexpr uint32_t kFull = 0xffffffffu;
constexpr uint32_t kDenseStage = 0x100u;  // L[q] flag: dense superset (the fused pass stages stores)
#ifndef SUCO_FUSED_PPW
#define SUCO_FUSED_PPW 4
#endif
constexpr uint32_t kFusedPPW = SUCO_FUSED_PPW;  // pieces per warp in the fused pass (large batches)

__device__ __forceinline__ void fadd(uint32_t a, uint32_t b, uint32_t c, uint32_t& s, uint32_t& cy) {
    s = a ^ b ^ c;
    cy = (a & b) | (c & (a ^ b));
}

// 32x32 bit transpose across a warp: row r = lane (bit c = column c) ->
// lane c holds column c (bit r = row r). Five butterfly stages; the byte
// stages (16, 8) are one PRMT with a per-lane selector, the bit stages
// (4, 2, 1) a rotate by a per-lane amount and one LOP3 with a per-lane mask
// (bits that wrap around land only where the mask keeps x).
struct Xpose {
    uint32_t sel16, sel8, amt4, amt2, amt1, msk4, msk2, msk1;
    __device__ explicit Xpose(uint32_t lane) {
        sel16 = (lane & 16) ? 0x3276u : 0x5410u;
        sel8 = (lane & 8) ? 0x3715u : 0x6240u;
        amt4 = (lane & 4) ? 28u : 4u;
        amt2 = (lane & 2) ? 30u : 2u;
        amt1 = (lane & 1) ? 31u : 1u;
        msk4 = (lane & 4) ? ~0x0f0f0f0fu : 0x0f0f0f0fu;
        msk2 = (lane & 2) ? ~0x33333333u : 0x33333333u;
        msk1 = (lane & 1) ? ~0x55555555u : 0x55555555u;
        // opaque copies: ptxas would otherwise rematerialise the per-lane constants inside the
        // scoring loops (S2R + R2P + SELs per tile, measured in the cfg4 fused pass's SASS)
        pin(sel16), pin(sel8), pin(amt4), pin(amt2), pin(amt1), pin(msk4), pin(msk2), pin(msk1);
    }
    __device__ __forceinline__ static void pin(uint32_t& v) { asm volatile("mov.b32 %0, %0;" : "+r"(v)); }
    __device__ __forceinline__ static uint32_t bits(uint32_t x, uint32_t y, uint32_t amt, uint32_t msk) {
        const uint32_t r = __funnelshift_l(y, y, amt);
        return (x & msk) | (r & ~msk);
    }
    __device__ __forceinline__ uint32_t operator()(uint32_t x) const {
        x = __byte_perm(x, __shfl_xor_sync(kFull, x, 16), sel16);
        x = __byte_perm(x, __shfl_xor_sync(kFull, x, 8), sel8);
        x = bits(x, __shfl_xor_sync(kFull, x, 4), amt4, msk4);
        x = bits(x, __shfl_xor_sync(kFull, x, 2), amt2, msk2);
        x = bits(x, __shfl_xor_sync(kFull, x, 1), amt1, msk1);
        return x;
    }
};

// Bit-sliced x >= t over 32 NP-bit numbers (planes B[0..NP)), t in [0, 2^NP + 1].
template <uint32_t NP>
__device__ __forceinline__ uint32_t ge_mask_n(const uint32_t (&B)[NP], uint32_t t) {
    if (t >> NP) return 0u;  // above every representable score
    uint32_t gt = 0, eq = kFull;
#pragma unroll
    for (int i = NP - 1; i >= 0; --i) {
        const uint32_t tm = ((t >> i) & 1u) ? kFull : 0u;
        gt |= eq & B[i] & ~tm;
        eq &= ~(B[i] ^ tm);
    }
    return gt | eq;
}

// Up to 8 subspaces: one uint4 of u16 codes per point (NC = 1, 4 score planes); up to 16: two
// (NC = 2, 5 planes).
template <uint32_t NC>
struct Np {
    static constexpr uint32_t v = NC == 1 ? 4 : 5;
};
template <uint32_t NC>
struct Codes {
    uint4 v[NC];
};

// Masks of the CTA's query block (32*W queries): W words per (subspace, cell)
// slot; bit j of word w <=> query q0 + 32w + j retrieved (s, cell).
template <uint32_t kDT, uint32_t W>
__device__ void build_masks(const DenseArgs& a, uint32_t* M, uint64_t q0, uint32_t nqb) {
    constexpr uint32_t kDW = kDT / 32;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t words = (dense_none(a.ns, a.K) + 1) * W;
    for (uint32_t i = tid; i < words; i += kDT) M[i] = 0;
    __syncthreads();
    for (uint32_t j = warp; j < nqb; j += kDW) {
        const uint64_t q = a.qmap ? a.qmap[q0 + j] : q0 + j;
        for (uint32_t s = 0; s < a.ns; ++s) {
            const uint64_t t = q * a.ns + s;
            const uint32_t cnt = a.cells_off ? static_cast<uint32_t>(a.cells_off[t + 1] - a.cells_off[t]) : a.ncells[t];
            const uint32_t* cp = a.cells + (a.cells_off ? a.cells_off[t] : t * a.cells_cap);
            for (uint32_t i = lane; i < cnt; i += 32)
                atomicOr(M + dense_slot(a.ns, a.K, s, cp[i]) * W + (j >> 5), 1u << (j & 31u));
        }
    }
    __syncthreads();
}

template <uint32_t W>
__device__ __forceinline__ void mask_at(const uint32_t* M, uint32_t slot, uint32_t (&m)[W]) {
    if constexpr (W == 1) {
        m[0] = M[slot];
    } else {
        const uint2 v = reinterpret_cast<const uint2*>(M)[slot];
        m[0] = v.x;
        m[1] = v.y;
    }
}

// Bit-planes of the scores of the 32 points [t0, t0 + 32) (lane = point t0 + lane) for the
// block's 32*W queries: b[w][i] bit j = bit i of query (32w + j)'s score.
template <uint32_t NC>
__device__ __forceinline__ Codes<NC> load_codes(const DenseArgs& a, uint64_t p, uint64_t p_hi) {
    const uint32_t none = dense_none(a.ns, a.K);
    Codes<NC> c;
#pragma unroll
    for (uint32_t i = 0; i < NC; ++i) c.v[i] = make_uint4(none | (none << 16), none | (none << 16), none | (none << 16), none | (none << 16));
    if (p < p_hi) {
#pragma unroll
        for (uint32_t i = 0; i < NC; ++i) c.v[i] = __ldg(a.codes + p * NC + i);
    }
    return c;
}

template <uint32_t NC>
__device__ __forceinline__ Codes<NC> load_codes_at(const DenseArgs& a, const uint4* p, bool valid) {
    const uint32_t none = dense_none(a.ns, a.K);
    const uint32_t nn = none | (none << 16);
    Codes<NC> c;
#pragma unroll
    for (uint32_t i = 0; i < NC; ++i) c.v[i] = valid ? __ldg(p + i) : make_uint4(nn, nn, nn, nn);
    return c;
}

// One 32-bit mask per slot at the shared-window address mb + 4 slot: the shift and add are one LEA
// per lookup (through a generic pointer ptxas adds the window base to every address separately).
// MB >= 0: the table's shared-window address is the constant MB (checked by the caller), folded
// into the load's immediate offset: the lookup's address is then one shift-and-mask of the code.
template <int MB>
__device__ __forceinline__ uint32_t lds_slot(uint32_t mb, uint32_t slot) {
    uint32_t v;
    if constexpr (MB >= 0) {
        asm volatile("ld.shared.b32 %0, [%1+%2];" : "=r"(v) : "r"(slot << 2), "n"(MB));
    } else {
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(mb + (slot << 2)));
    }
    return v;
}

template <uint32_t W, uint32_t NC, int MB = -1>
__device__ __forceinline__ void masks_of(const uint32_t* M, const Codes<NC>& c, uint32_t (&m)[8 * NC][W]) {
    if constexpr (W == 1) {
        const uint32_t mb = static_cast<uint32_t>(__cvta_generic_to_shared(M));
#pragma unroll
        for (uint32_t i = 0; i < NC; ++i) {
            m[8 * i + 0][0] = lds_slot<MB>(mb, c.v[i].x & 0xffffu);
            m[8 * i + 1][0] = lds_slot<MB>(mb, c.v[i].x >> 16);
            m[8 * i + 2][0] = lds_slot<MB>(mb, c.v[i].y & 0xffffu);
            m[8 * i + 3][0] = lds_slot<MB>(mb, c.v[i].y >> 16);
            m[8 * i + 4][0] = lds_slot<MB>(mb, c.v[i].z & 0xffffu);
            m[8 * i + 5][0] = lds_slot<MB>(mb, c.v[i].z >> 16);
            m[8 * i + 6][0] = lds_slot<MB>(mb, c.v[i].w & 0xffffu);
            m[8 * i + 7][0] = lds_slot<MB>(mb, c.v[i].w >> 16);
        }
        return;
    }
#pragma unroll
    for (uint32_t i = 0; i < NC; ++i) {
        mask_at<W>(M, c.v[i].x & 0xffffu, m[8 * i + 0]);
        mask_at<W>(M, c.v[i].x >> 16, m[8 * i + 1]);
        mask_at<W>(M, c.v[i].y & 0xffffu, m[8 * i + 2]);
        mask_at<W>(M, c.v[i].y >> 16, m[8 * i + 3]);
        mask_at<W>(M, c.v[i].z & 0xffffu, m[8 * i + 4]);
        mask_at<W>(M, c.v[i].z >> 16, m[8 * i + 5]);
        mask_at<W>(M, c.v[i].w & 0xffffu, m[8 * i + 6]);
        mask_at<W>(M, c.v[i].w >> 16, m[8 * i + 7]);
    }
}

// The carry-save adder tree over a point's 8 * NC masks: its score bit-planes for the block.
template <uint32_t W, uint32_t NC>
__device__ __forceinline__ void csa_planes(const uint32_t (&m)[8 * NC][W], uint32_t (&b)[W][Np<NC>::v]) {
#pragma unroll
    for (uint32_t w = 0; w < W; ++w) {
        if constexpr (NC == 1) {
            uint32_t s1, c1, s2, c2, b0, c4, s5, c5;
            fadd(m[0][w], m[1][w], m[2][w], s1, c1);
            fadd(m[3][w], m[4][w], m[5][w], s2, c2);
            const uint32_t s3 = m[6][w] ^ m[7][w], c3 = m[6][w] & m[7][w];
            fadd(s1, s2, s3, b0, c4);  // weight 1
            fadd(c1, c2, c3, s5, c5);  // weight 2 (+ carry weight 4)
            const uint32_t c6 = s5 & c4;
            b[w][0] = b0;
            b[w][1] = s5 ^ c4;
            b[w][2] = c5 ^ c6;
            b[w][3] = c5 & c6;
        } else {  // 16 inputs -> 5 planes (carry-save tree)
            uint32_t s1, c1, s2, c2, s3, c3, s4, c4, s5, c5, t1, d1, t2, d2, u1, e1, u2, e2, u3, e3, v1, f1;
            fadd(m[0][w], m[1][w], m[2][w], s1, c1);
            fadd(m[3][w], m[4][w], m[5][w], s2, c2);
            fadd(m[6][w], m[7][w], m[8][w], s3, c3);
            fadd(m[9][w], m[10][w], m[11][w], s4, c4);
            fadd(m[12][w], m[13][w], m[14][w], s5, c5);
            fadd(s1, s2, s3, t1, d1);  // weight 1
            fadd(s4, s5, m[15][w], t2, d2);
            const uint32_t d3 = t1 & t2;
            b[w][0] = t1 ^ t2;
            fadd(c1, c2, c3, u1, e1);  // weight 2
            fadd(c4, c5, d1, u2, e2);
            fadd(d2, d3, u1, u3, e3);
            const uint32_t e4 = u2 & u3;
            b[w][1] = u2 ^ u3;
            fadd(e1, e2, e3, v1, f1);  // weight 4
            const uint32_t f2 = v1 & e4;
            b[w][2] = v1 ^ e4;
            b[w][3] = f1 ^ f2;  // weight 8
            b[w][4] = f1 & f2;  // weight 16
        }
    }
}

template <uint32_t W, uint32_t NC>
__device__ __forceinline__ void planes_of(const uint32_t* M, const Codes<NC>& c, uint32_t (&b)[W][Np<NC>::v]) {
    uint32_t m[8 * NC][W];
    masks_of<W, NC>(M, c, m);
    csa_planes<W, NC>(m, b);
}

// The same scores with lane = query (word w: query 32w + lane): planes B[w][*] (bit r =
// point t0 + r).
template <uint32_t W, uint32_t NC>
__device__ __forceinline__ void score_tile(const DenseArgs& a, const uint32_t* M, uint64_t t0, uint64_t p_hi,
                                           const Xpose& xp, uint32_t (&B)[W][Np<NC>::v], uint32_t lane) {
    uint32_t b[W][Np<NC>::v];
    planes_of<W, NC>(M, load_codes<NC>(a, t0 + lane, p_hi), b);
#pragma unroll
    for (uint32_t w = 0; w < W; ++w) {
#pragma unroll
        for (uint32_t i = 0; i < Np<NC>::v; ++i) B[w][i] = xp(b[w][i]);
    }
}

// K1: per (query, piece) #points with score >= t, t = 1..8*NC (u16 each, NC uint4 per row).
template <uint32_t kDT, uint32_t W, uint32_t NC>
__global__ void __launch_bounds__(kDT, 1024 / kDT) dense_hist_kernel(DenseArgs a) {
    constexpr uint32_t kDW = kDT / 32, NP = Np<NC>::v, LV = 8 * NC;
    extern __shared__ uint32_t M[];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint64_t q0 = uint64_t(blockIdx.x) * 32 * W;
    const uint64_t nvalid = a.qmap ? *a.nmap : a.nq;  // fallback run: only the listed queries
    if (q0 >= nvalid) return;
    const uint32_t nqb = static_cast<uint32_t>(min_u64(32 * W, nvalid - q0));
    build_masks<kDT, W>(a, M, q0, nqb);
    const uint32_t row = blockIdx.y * kDW + warp;  // histogram row
    if (row >= a.P) return;
    const uint64_t lo = uint64_t(row) * (a.pstride ? a.pstride : 1u) * a.WP;  // its piece (a sample when pstride > 1)
    if (lo >= a.n) return;
    const uint64_t hi = min_u64(a.n, lo + a.WP);
    const uint32_t piece = row;
    uint32_t cnt[W][LV];
#pragma unroll
    for (uint32_t w = 0; w < W; ++w) {
#pragma unroll
        for (uint32_t t = 0; t < LV; ++t) cnt[w][t] = 0;
    }
    const Xpose xp(lane);
    for (uint64_t t0 = lo; t0 < hi; t0 += 32) {
        uint32_t B[W][NP];
        score_tile<W, NC>(a, M, t0, hi, xp, B, lane);
        // points past `hi` score 0: they never count for t >= 1
#pragma unroll
        for (uint32_t w = 0; w < W; ++w) {
            if constexpr (NC == 1) {
                const uint32_t B0 = B[w][0], B1 = B[w][1], B2 = B[w][2], B3 = B[w][3];
                const uint32_t g8 = B3, g4 = B3 | B2, g2 = g4 | B1, g1 = g2 | B0;
                const uint32_t g6 = B3 | (B2 & B1), g5 = B3 | (B2 & (B1 | B0)), g7 = B3 | (B2 & B1 & B0);
                const uint32_t g3 = g4 | (B1 & B0);
                cnt[w][0] += __popc(g1);
                cnt[w][1] += __popc(g2);
                cnt[w][2] += __popc(g3);
                cnt[w][3] += __popc(g4);
                cnt[w][4] += __popc(g5);
                cnt[w][5] += __popc(g6);
                cnt[w][6] += __popc(g7);
                cnt[w][7] += __popc(g8);
            } else {  // #(score == v), v = 1..16; suffix sums at the end
#pragma unroll
                for (uint32_t v = 1; v <= LV; ++v) {
                    uint32_t e = kFull;
#pragma unroll
                    for (uint32_t i = 0; i < NP; ++i) e &= ((v >> i) & 1u) ? B[w][i] : ~B[w][i];
                    cnt[w][v - 1] += __popc(e);
                }
            }
        }
    }
#pragma unroll
    for (uint32_t w = 0; w < W; ++w) {
        if constexpr (NC != 1) {
#pragma unroll
            for (int t = LV - 2; t >= 0; --t) cnt[w][t] += cnt[w][t + 1];
        }
        if (32 * w + lane < nqb) {
            const uint64_t q = a.qmap ? a.qmap[q0 + 32 * w + lane] : q0 + 32 * w + lane;
#pragma unroll
            for (uint32_t i = 0; i < NC; ++i) {
                uint4 v;
                v.x = cnt[w][8 * i + 0] | (cnt[w][8 * i + 1] << 16);
                v.y = cnt[w][8 * i + 2] | (cnt[w][8 * i + 3] << 16);
                v.z = cnt[w][8 * i + 4] | (cnt[w][8 * i + 5] << 16);
                v.w = cnt[w][8 * i + 6] | (cnt[w][8 * i + 7] << 16);
                reinterpret_cast<uint4*>(a.hist)[(q * a.P + piece) * NC + i] = v;
            }
        }
    }
}

__device__ __forceinline__ uint32_t level(const uint4& v, uint32_t t) {  // #score >= t, t in 1..8
    const uint32_t w = t <= 2 ? v.x : t <= 4 ? v.y : t <= 6 ? v.z : v.w;
    return (t & 1u) ? (w & 0xffffu) : (w >> 16);
}

// #score >= t, t in 1..8*nc, from a histogram row of nc uint4
__device__ __forceinline__ uint32_t level_n(const uint4* row, uint32_t t) {
    return level(row[(t - 1) >> 3], ((t - 1) & 7u) + 1);
}

__device__ __forceinline__ uint32_t nc_of(const DenseArgs& a) { return a.nc ? a.nc : 1u; }

// The global piece index of local piece p (tie cuts are in global id order; block-cyclic shards).
__device__ __forceinline__ uint32_t gpiece(const DenseArgs& a, uint32_t p) {
    return a.shG ? ((p / a.shPPB) * a.shG + a.shR) * a.shPPB + p % a.shPPB : p;
}

// Which single-pass compaction kernel takes query q: the warp kernel for dense supersets (the L[q]
// flag of the bound kernel), the thread kernel for sparse ones (Tuning::dense_compact forces either).
__device__ __forceinline__ bool dense_compact_warp(const DenseArgs& a, uint64_t q) {
    return a.compact_mode == 2 || (a.compact_mode == 0 && (a.L[q] & kDenseStage));
}

// Single-pass candidate buffers, [query][piece][B]: entry e of (q, piece) at cb_base(q, piece) +
// cb_off(e); a lane of the fused pass appends to its own contiguous buffer. (Measured against a
// [query][chunk][piece] interleave at cfg4: the interleave wrote 5.7 GB instead of 4.4 GB.)
__device__ __forceinline__ uint16_t* cb_base(const DenseArgs& a, uint64_t q, uint32_t piece) {
    return a.cbuf + (q * a.P + piece) * a.B;
}
__device__ __forceinline__ uint32_t cb_off(const DenseArgs&, uint32_t e) { return e; }

// K2: warp per query — T, need, per-piece tie quota (id order) and output offset.
__global__ void __launch_bounds__(256) dense_plan_kernel(DenseArgs a) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t qi = uint64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (qi >= (a.qmap ? *a.nmap : a.nq)) return;
    const uint64_t q = a.qmap ? a.qmap[qi] : qi;
    const uint32_t nc = nc_of(a), LV = 8 * nc;
    const uint4* h = reinterpret_cast<const uint4*>(a.hist) + q * a.P * nc;
    uint32_t tot[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) tot[t] = 0;
    for (uint32_t p = lane; p < a.P; p += 32) {
#pragma unroll
        for (uint32_t t = 1; t <= 16; ++t) {
            if (t <= LV) tot[t - 1] += level_n(h + p * nc, t);
        }
    }
#pragma unroll
    for (int t = 0; t < 16; ++t) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) tot[t] += __shfl_xor_sync(kFull, tot[t], o);
    }
    uint32_t T = 0;
#pragma unroll
    for (int t = 16; t >= 1; --t) {
        if (T == 0 && static_cast<uint32_t>(t) <= min(a.ns, LV) && tot[t - 1] >= a.m) T = t;
    }
    uint32_t gtT = 0;
#pragma unroll
    for (int t = 1; t <= 16; ++t) {
        if (static_cast<uint32_t>(t) == T + 1 && static_cast<uint32_t>(t) <= LV) gtT = tot[t - 1];
    }
    const uint64_t need = a.m - gtT;
    uint64_t ties_run = 0, out_run = 0;
    for (uint32_t p0 = 0; p0 < a.P; p0 += 32) {
        const uint32_t p = p0 + lane;
        uint32_t ties = 0, gt = 0;
        if (p < a.P) {
            const uint32_t len = static_cast<uint32_t>(min_u64(a.WP, a.n - uint64_t(p) * a.WP));
            const uint32_t geT = T ? level_n(h + p * nc, T) : len;
            gt = T + 1 <= LV ? level_n(h + p * nc, T + 1) : 0u;
            ties = geT - gt;
        }
        uint32_t tx = ties;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, tx, o);
            if (lane >= static_cast<uint32_t>(o)) tx += y;
        }
        const uint32_t tsum = __shfl_sync(kFull, tx, 31);
        const uint64_t before = ties_run + tx - ties;
        const uint32_t quota = before >= need ? 0u : static_cast<uint32_t>(min_u64(ties, need - before));
        const uint32_t take = gt + quota;
        uint32_t ox = take;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, ox, o);
            if (lane >= static_cast<uint32_t>(o)) ox += y;
        }
        const uint32_t osum = __shfl_sync(kFull, ox, 31);
        if (p < a.P) {
            a.quota[q * a.P + p] = quota;
            a.base[q * a.P + p] = static_cast<uint32_t>(out_run + ox - take);

        }
        ties_run += tsum;
        out_run += osum;
    }
    if (lane == 0) a.T[q] = T;
}

// Single-pass plan: T == L exactly when #(score >= L) >= m > #(score >= L+1); then the quotas and
// offsets come from those two levels; otherwise the query is flagged for the exact fallback.
__global__ void __launch_bounds__(256) dense_plan_fused_kernel(DenseArgs a) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t q = uint64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (q >= a.nq) return;
    const uint32_t* h = a.h2 + q * a.P;
    uint64_t geL1 = 0;  // #(score > L)
    for (uint32_t p = lane; p < a.P; p += 32) geL1 += h[p] >> 16;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) geL1 += __shfl_xor_sync(kFull, geL1, o);
    const uint32_t L = a.L[q] & 0xffu;
    // (#(score >= L) >= m is checked below as: the ties counted before the cut cover `need`; pieces
    // past every tie cut of their block record #(score > L) in both halves)
    bool ok = L >= 1 && geL1 < a.m;
    const uint64_t need = a.m - geL1;
    uint64_t ties_run = 0, gt_run = 0, tie_run = 0;
    for (uint32_t p0 = 0; p0 < a.P; p0 += 32) {
        const uint32_t p = p0 + lane;
        uint32_t ties = 0, gt = 0;
        if (p < a.P) {
            const uint32_t v = h[p];
            gt = v >> 16;
            ties = (v & 0xffffu) - gt;
        }
        uint32_t tx = ties;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, tx, o);
            if (lane >= static_cast<uint32_t>(o)) tx += y;
        }
        const uint32_t tsum = __shfl_sync(kFull, tx, 31);
        const uint64_t before = ties_run + tx - ties;
        const uint32_t quota = before >= need ? 0u : static_cast<uint32_t>(min_u64(ties, need - before));
        const uint32_t take = gt + quota;
        // offsets: score > T entries from 0 in piece order, then the ties from #(score > T) = m - need
        uint32_t gx = gt, qx = quota;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, gx, o), z = __shfl_up_sync(kFull, qx, o);
            if (lane >= static_cast<uint32_t>(o)) {
                gx += y;
                qx += z;
            }
        }
        const uint32_t gsum = __shfl_sync(kFull, gx, 31), qsum = __shfl_sync(kFull, qx, 31);
        if (p < a.P) {
            a.quota[q * a.P + p] = quota;
            a.base[q * a.P + p] = static_cast<uint32_t>(gt_run + gx - gt);
            a.base2[q * a.P + p] = static_cast<uint32_t>(geL1 + tie_run + qx - quota);
            if (take && a.ccnt[q * a.P + p] > a.B) ok = false;  // a contributing buffer overflowed
            if (quota && a.pcut && p >= a.pcut[q]) ok = false;   // ties needed past the tie cut
        }
        ties_run += tsum;
        gt_run += gsum;
        tie_run += qsum;
    }
    ok = __all_sync(kFull, ok) && ties_run >= need;
    if (lane == 0) {
        a.qflag[q] = ok ? 0u : 1u;
        if (ok && a.clist) {  // the compaction kernels' work lists
            const uint32_t wl = dense_compact_warp(a, q) ? 0u : 1u;
            a.clist[wl * a.nq + atomicAdd(a.nclist + wl, 1u)] = static_cast<uint32_t>(q);
        }
        a.T[q] = L;
    }
}

// K3: re-score each piece; lane = query emits score > T and the first quota ties (id order).
template <uint32_t kDT, uint32_t W, uint32_t NC>
__global__ void __launch_bounds__(kDT, 1024 / kDT) dense_emit_kernel(DenseArgs a) {
    constexpr uint32_t kDW = kDT / 32, NP = Np<NC>::v;
    extern __shared__ uint32_t M[];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint64_t q0 = uint64_t(blockIdx.x) * 32 * W;
    const uint64_t nvalid = a.qmap ? *a.nmap : a.nq;  // fallback run: only the listed queries
    if (q0 >= nvalid) return;
    const uint32_t nqb = static_cast<uint32_t>(min_u64(32 * W, nvalid - q0));
    build_masks<kDT, W>(a, M, q0, nqb);
    const uint32_t piece = blockIdx.y * kDW + warp;
    if (piece >= a.P) return;
    const uint64_t lo = uint64_t(piece) * a.WP;
    const uint64_t hi = min_u64(a.n, lo + a.WP);
    bool mine[W];
    uint32_t T[W], quota[W], pos[W], tseen[W];
    uint32_t* out[W];
#pragma unroll
    for (uint32_t w = 0; w < W; ++w) {
        mine[w] = 32 * w + lane < nqb;
        const uint64_t q = !mine[w] ? 0 : a.qmap ? a.qmap[q0 + 32 * w + lane] : q0 + 32 * w + lane;
        T[w] = mine[w] ? a.T[q] : 0u;
        quota[w] = mine[w] ? a.quota[q * a.P + piece] : 0u;
        pos[w] = mine[w] ? a.base[q * a.P + piece] : 0u;
        tseen[w] = 0;
        out[w] = a.cands + (mine[w] ? q : 0) * a.m;
    }
    const Xpose xp(lane);
    for (uint64_t t0 = lo; t0 < hi; t0 += 32) {
        uint32_t B[W][NP];
        score_tile<W, NC>(a, M, t0, hi, xp, B, lane);
        const uint32_t vmask = hi - t0 >= 32 ? kFull : ((1u << (hi - t0)) - 1u);
        if (a.scores_dbg && q0 == 0 && lane == 0 && mine[0]) {  // parity dump: query 0's scores
            for (uint32_t r = 0; r < 32 && t0 + r < hi; ++r) {
                uint32_t sc = 0;
#pragma unroll
                for (uint32_t i = 0; i < NP; ++i) sc |= ((B[0][i] >> r) & 1u) << i;
                a.scores_dbg[t0 + r] = static_cast<uint8_t>(sc);
            }
        }
#pragma unroll
        for (uint32_t w = 0; w < W; ++w) {
            if (!mine[w]) continue;  // lanes past the block's last query only feed the transposes
            const uint32_t geT = ge_mask_n<NP>(B[w], T[w]) & vmask;
            const uint32_t gt = ge_mask_n<NP>(B[w], T[w] + 1) & vmask;
            const uint32_t eq = geT & ~gt;
            uint32_t take = gt;
            if (eq && tseen[w] < quota[w]) {
                const uint32_t r = quota[w] - tseen[w];
                uint32_t rest = eq;
                for (uint32_t i = 0; i < r && rest; ++i) rest &= rest - 1;  // drop the first r ties
                take |= eq ^ rest;
            }
            tseen[w] += __popc(eq);
            while (take) {
                const uint32_t b = __ffs(take) - 1;
                take &= take - 1;
                __stcs(out[w] + pos[w]++, static_cast<uint32_t>(t0) + b);
            }
        }
    }
}

// K0 -> L: per query, the largest t whose sampled #(score >= t), scaled to n, reaches m (0 if none).
// L (the speculative T), the dense-superset flag and the tie cut of one query from its sampled
// totals tot[t - 1] = #(score >= t) over `sampled` points of a corpus of n points in P pieces.
struct Bound {
    uint32_t L, cut;
    bool dense;
};
__device__ __forceinline__ Bound bound_core(const DenseArgs& a, const uint32_t (&tot)[16], uint64_t sampled,
                                            uint64_t n, uint32_t P) {
    const uint32_t LV = 8 * nc_of(a);
    uint32_t L = 0;
    uint32_t atL = 0;
#pragma unroll
    for (int t = 16; t >= 1; --t) {
        if (L == 0 && static_cast<uint32_t>(t) <= min(a.ns, LV) && sampled &&
            static_cast<double>(tot[t - 1]) * static_cast<double>(n) / static_cast<double>(sampled) >=
                static_cast<double>(a.m)) {
            L = t;
            atL = tot[t - 1];
        }
    }
    // The single pass writes one 8-byte record per tile holding a point with score >= L, at most
    // 0.25 B per (point, query) even when every tile has one; a second scoring pass costs more.
    // dense supersets (> 1% of the points at L) make the fused pass stage its stores
    const bool dense = L && (a.stage_all || static_cast<double>(atL) > 0.01 * static_cast<double>(sampled));
    // Tie cut: the quota takes the first `need` score == L points in id order, so the fused pass
    // stores tie entries only in the pieces the quota is expected to reach (x1.25 + 8 pieces of
    // margin); later pieces keep just their score > L entries. A quota that reaches past the cut
    // flags the query for the exact fallback.
    uint32_t cut = P;
    if (L && sampled && a.pcut && !a.no_cut) {
        uint32_t above = 0;  // sampled #(score >= L + 1)
#pragma unroll
        for (int t = 1; t <= 16; ++t) {
            if (static_cast<uint32_t>(t) == L + 1 && static_cast<uint32_t>(t) <= LV) above = tot[t - 1];
        }
        const double scale = static_cast<double>(n) / static_cast<double>(sampled);
        const double ties = (static_cast<double>(atL) - static_cast<double>(above)) * scale;
        const double need = static_cast<double>(a.m) - static_cast<double>(above) * scale;
        if (ties > 0.0 && need < ties) {
            const double cs = a.cut_scale > 0.f ? static_cast<double>(a.cut_scale) : 1.25;
            // (+8 pieces of 2048 points: the pad is in points, whatever the piece size)
            const double cp = a.cut_scale > 0.f ? static_cast<double>(a.cut_pad) : 8.0 * kDensePiece / a.WP;
            const double c = static_cast<double>(P) * (need > 0.0 ? need / ties : 0.0) * cs + cp;
            cut = c < static_cast<double>(P) ? static_cast<uint32_t>(c) : P;
        }
    }
    return {L, cut, dense};
}

// The sampled totals of one query (warp): tot[t - 1] = #(score >= t) over the sampled pieces, and
// the number of points they scanned.
__device__ __forceinline__ uint64_t sample_totals(const DenseArgs& a, uint64_t q, uint32_t lane, uint32_t (&tot)[16]) {
    const uint32_t nc = nc_of(a), LV = 8 * nc;
    const uint4* h = reinterpret_cast<const uint4*>(a.hsample) + q * a.Ps * nc;
#pragma unroll
    for (int t = 0; t < 16; ++t) tot[t] = 0;
    for (uint32_t p = lane; p < a.Ps; p += 32) {
#pragma unroll
        for (uint32_t t = 1; t <= 16; ++t) {
            if (t <= LV) tot[t - 1] += level_n(h + p * nc, t);
        }
    }
#pragma unroll
    for (int t = 0; t < 16; ++t) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) tot[t] += __shfl_xor_sync(kFull, tot[t], o);
    }
    uint64_t sampled = 0;  // points the sample scanned
    const uint32_t swp = a.sWP ? a.sWP : a.WP;
    for (uint32_t p = 0; p < a.Ps; ++p) {
        const uint64_t lo = uint64_t(p) * a.pstride * swp;
        if (lo < a.n) sampled += min_u64(swp, a.n - lo);
    }
    return sampled;
}

__global__ void __launch_bounds__(256) dense_bound_kernel(DenseArgs a) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t q = uint64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (q >= a.nq) return;
    uint32_t tot[16];
    const uint64_t sampled = sample_totals(a, q, lane, tot);
    const Bound b = bound_core(a, tot, sampled, a.n, a.P);
    if (lane == 0) {
        a.L[q] = b.L | (b.dense ? kDenseStage : 0u);
        if (a.pcut) a.pcut[q] = b.cut;
    }
}

// The fused pass's walk over a warp's pieces (below). STAGE: entries go through a 64-bit register
// (four per 8-byte store) — for dense supersets, where 2-byte stores multiply DRAM traffic; sparse
// ones store each entry directly (fewer instructions per tile).
template <uint32_t kDW, uint32_t W, bool STAGE, uint32_t NC, int MB = -1>
__device__ __forceinline__ void fused_pieces(const DenseArgs& a, const uint32_t* M, uint64_t q0, uint32_t nqb,
                                             const uint32_t (&TL)[W][Np<NC>::v], const uint32_t (&live)[W],
                                             const uint32_t (&cut)[W], uint32_t lane, uint32_t warp) {
    constexpr uint32_t NP = Np<NC>::v;
    const Xpose xp(lane);
    // a warp walks ppw consecutive pieces: the masks are built once per CTA for them all
    for (uint32_t k = 0; k < a.ppw; ++k) {
        const uint32_t piece = (blockIdx.y * kDW + warp) * a.ppw + k;
        if (piece >= a.P) return;
        const uint64_t lo = uint64_t(piece) * a.WP;
        const uint64_t hi = min_u64(a.n, lo + a.WP);
        uint32_t cnt[W], nb[W];
        uint16_t* bp[W];  // [query][piece][B]: a lane appends to its own contiguous buffer (next store)
        uint64_t sw[W];   // STAGE: four entries shifted in from the top
#pragma unroll
        for (uint32_t w = 0; w < W; ++w) {
            cnt[w] = 0;
            nb[w] = 0;
            sw[w] = 0;
            const uint64_t q = 32 * w + lane < nqb ? q0 + 32 * w + lane : q0;  // idle lanes append nothing
            bp[w] = cb_base(a, q, piece);
        }
        // 32-bit tile loop over the piece: a running code pointer, the piece's point count
        const uint32_t len = static_cast<uint32_t>(hi - lo);
        const uint4* cptr = a.codes + (lo + lane) * NC;
        // software pipeline: the next tile's mask lookups are in flight while this tile's planes
        // are compared, transposed and emitted; its codes were loaded a tile before that
        uint32_t mk[8 * NC][W];
        // (unconditional loads: the code rows are padded with zero-slot codes past n, and loads past
        // a piece's end read the next piece's codes, never scored)
        masks_of<W, NC, MB>(M, load_codes_at<NC>(a, cptr, true), mk);
        Codes<NC> code1 = load_codes_at<NC>(a, cptr + 32 * NC, true);
        // Pieces past every lane's tie cut need only score > L (lane = query): one transpose per tile
        // instead of two; their #(score >= L) is not needed by the plan (its ties are never taken:
        // a quota that reaches past the cut flags the query) and is recorded as #(score > L).
        bool need_ge = false;
        const uint32_t gp = gpiece(a, piece);
#pragma unroll
        for (uint32_t w = 0; w < W; ++w) need_ge |= gp < cut[w];
        need_ge = __any_sync(kFull, need_ge);
        // the tile loop, compiled once for pieces some query of the block still needs ties from
        // (NEED_GE) and once for pieces past every tie cut
        auto tile_loop = [&](auto need_ge_c) {
            constexpr bool NEED_GE = decltype(need_ge_c)::value;
            for (uint32_t tb = 0; tb < len; tb += 32) {
                cptr += 32 * NC;
                // two tiles ahead: the code loads miss L2 often enough that one tile did not cover them
                const Codes<NC> next = load_codes_at<NC>(a, cptr + 32 * NC, true);
                uint32_t b[W][NP];
                csa_planes<W, NC>(mk, b);
                masks_of<W, NC, MB>(M, code1, mk);  // (past the piece end: the zero slot)
                code1 = next;
    #pragma unroll
                for (uint32_t w = 0; w < W; ++w) {
                    // most significant plane first; points past the piece end score 0 < L
                    uint32_t gt = b[w][NP - 1] & ~TL[w][NP - 1], eq = ~(b[w][NP - 1] ^ TL[w][NP - 1]);
    #pragma unroll
                    for (int i = NP - 2; i >= 0; --i) {
                        gt |= eq & b[w][i] & ~TL[w][i];
                        eq &= ~(b[w][i] ^ TL[w][i]);
                    }
                    if constexpr (!NEED_GE) {
                        // Past every tie cut only score > L entries are kept, and they are sparse; their order
                        // is free (the plan and the compaction keep every one), so no transpose: each point
                        // (lane) holding some, in turn, broadcasts its query mask and those queries' lanes
                        // append it.
                        // Branch-free: every lane runs the warp-uniform loop, the hit lane stores (one
                        // predicated 2-byte store at its entry count; such pieces never stage).
                        const uint32_t gl = gt & live[w];  // lane = point, bit j = query 32w + j
                        uint32_t pending = __ballot_sync(kFull, gl != 0);
                        while (pending) {
                            const uint32_t p = __ffs(pending) - 1;
                            pending &= pending - 1;
                            const uint32_t hit = (__shfl_sync(kFull, gl, p) >> lane) & 1u;
                            if (hit && nb[w] < a.B) bp[w][nb[w]] = static_cast<uint16_t>((tb + p) | 0x8000u);
                            nb[w] += hit;  // (#(score >= L) and #(score > L) are recorded alike: nb, after the loop)
                        }
                        continue;
                    }
                    const uint32_t g1 = xp(gt & live[w]);  // lane = query, bit r = point t0 + r
                    uint32_t bits = g1;
                    {
                        const uint32_t ge0 = xp((gt | eq) & live[w]);
                        cnt[w] += __popc(ge0) | (__popc(g1) << 16);
                        if (gp < cut[w]) bits = ge0;  // before the tie cut: every score >= L
                    }
                    if (bits) {  // id order; the capacity check once per tile while the buffer has room
                        const bool room = nb[w] + __popc(bits) <= a.B;
                        do {
                            const uint32_t r = __ffs(bits) - 1;
                            bits &= bits - 1;
                            if (room || nb[w] < a.B) {
                                const uint32_t v = (tb + r) | (((g1 >> r) & 1u) << 15);
                                if constexpr (STAGE) {
                                    sw[w] = (sw[w] >> 16) | (static_cast<uint64_t>(v) << 48);
                                    if ((nb[w] & 3u) == 3u) {
                                        *reinterpret_cast<uint64_t*>(bp[w]) = sw[w];
                                        bp[w] += 4;
                                    }
                                } else {
                                    *bp[w]++ = static_cast<uint16_t>(v);
                                }
                            }
                            ++nb[w];
                        } while (bits);
                    }
                }
            }
        };
        if (need_ge) {
            tile_loop(std::true_type{});
        } else {
            tile_loop(std::false_type{});
#pragma unroll
            for (uint32_t w = 0; w < W; ++w) cnt[w] = nb[w] * 0x10001u;  // every entry is a score > L point
        }
#pragma unroll
        for (uint32_t w = 0; w < W; ++w) {
            if (32 * w + lane < nqb) {
                const uint64_t i = (q0 + 32 * w + lane) * a.P + piece;
                if (STAGE && need_ge) {  // (pieces past every tie cut store each entry directly)
                    const uint32_t kept = min(nb[w], a.B), part = kept & 3u;
                    if (part)  // the last, partial chunk (at the running pointer): its entries down to the low end
                        *reinterpret_cast<uint64_t*>(bp[w]) = sw[w] >> (16 * (4 - part));
                }
                a.h2[i] = cnt[w];
                a.ccnt[i] = static_cast<uint16_t>(nb[w]);  // <= WP <= 32768
            }
        }
    }
}

// K3': one pass — the piece histograms (as K1) plus, per (query, piece), every point with
// score >= L[q] appended in id order to the pair's candidate buffer: the in-piece offset, bit 15
// set when the score is > L. A buffer holds B entries; a contributing piece that found more flags
// its query for the exact fallback.
template <uint32_t kDT, uint32_t W, uint32_t NC>
__global__ void __launch_bounds__(kDT, 1024 / kDT) dense_fused_kernel(DenseArgs a) {
    constexpr uint32_t kDW = kDT / 32, NP = Np<NC>::v;
    extern __shared__ uint32_t M[];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint64_t q0 = uint64_t(blockIdx.x) * 32 * W;
    const uint32_t nqb = static_cast<uint32_t>(min_u64(32 * W, a.nq - q0));
    const uint32_t myL = threadIdx.x < nqb ? a.L[q0 + threadIdx.x] : 0u;
    if (!__syncthreads_or((myL & 0xffu) != 0)) return;  // all two-pass
    const bool stage = __syncthreads_or(myL & kDenseStage);  // a dense superset in the block
    build_masks<kDT, W>(a, M, q0, nqb);
    // The bits of L[q] across the block's queries (word w, bit j = query 32w + j): one bit-sliced
    // comparison per tile, BEFORE the transpose (lane = point, bit = query), gives score > L and
    // score == L for all 32*W queries at once; only the two results are transposed (10 shuffles,
    // not 20 for the four planes). Counts per lane = query: #(score >= L) | #(score >= L+1) << 16.
    uint32_t TL[W][NP], live[W], cut[W];
#pragma unroll
    for (uint32_t w = 0; w < W; ++w) {
        const uint32_t L = 32 * w + lane < nqb ? a.L[q0 + 32 * w + lane] & 0xffu : 0u;  // 0: falls back
#pragma unroll
        for (uint32_t i = 0; i < NP; ++i) TL[w][i] = __ballot_sync(kFull, (L >> i) & 1u);
        live[w] = __ballot_sync(kFull, L != 0);
        cut[w] = a.pcut && 32 * w + lane < nqb ? a.pcut[q0 + 32 * w + lane] : a.P;
    }
    // the table at shared address 1024 (dynamic shared memory after the 1 KB reserved for the
    // system on sm_100): lookups with the base folded into the load's immediate
    const bool at1k = static_cast<uint32_t>(__cvta_generic_to_shared(M)) == 1024u;
    if (W == 1 && NC == 1 && at1k) {
        if (stage) fused_pieces<kDW, W, true, NC, 1024>(a, M, q0, nqb, TL, live, cut, lane, warp);
        else fused_pieces<kDW, W, false, NC, 1024>(a, M, q0, nqb, TL, live, cut, lane, warp);
    } else {
        if (stage) fused_pieces<kDW, W, true, NC>(a, M, q0, nqb, TL, live, cut, lane, warp);
        else fused_pieces<kDW, W, false, NC>(a, M, q0, nqb, TL, live, cut, lane, warp);
    }
}

// K4: thread per (query, piece), T == L: the piece's buffer holds its score >= T points in id
// order; keep every score > T entry and the first quota ties. A block takes 256 consecutive pieces
// of one query, whose outputs are two contiguous runs of the query's candidates (its score > T
// entries, its ties; pieces in order): each thread loads its whole buffer (independent 16-byte
// loads), places its kept ids in shared staging copies of the two runs, and the block writes the
// runs with coalesced stores. Runs longer than a staging half write their tail directly.
constexpr uint32_t kCompactStage = 4096;  // staged candidate ids per run (2 x 16 KB)
// DENSE: the dense-superset queries' pieces past their tie cut (score > T entries only, a few per
// piece: a thread each instead of a warp); else the sparse-superset queries' pieces.
template <bool DENSE>
__global__ void __launch_bounds__(256) dense_compact_thread_kernel(DenseArgs a) {
    __shared__ uint32_t stage[2][kCompactStage];
    __shared__ uint32_t run_lo[2], run_hi[2];
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t pbase = p * a.WP;
    const uint32_t nlist = a.nclist[DENSE ? 0 : 1];
    for (uint32_t j = blockIdx.y; j < nlist; j += gridDim.y) {
        const uint64_t q = DENSE ? a.clist[j] : a.clist[a.nq + j];  // an unflagged query of the list
        if constexpr (DENSE) {  // the whole block before the cut: the warp kernel has it
            if ((blockIdx.x + 1) * blockDim.x <= a.P && gpiece(a, (blockIdx.x + 1) * blockDim.x - 1) < a.pcut[q]) continue;
        }
        if (threadIdx.x < 2) {
            run_lo[threadIdx.x] = 0xffffffffu;
            run_hi[threadIdx.x] = 0;
        }
        __syncthreads();
        const uint64_t i = q * a.P + p;
        const bool mine = p < a.P && (!DENSE || gpiece(a, p) >= a.pcut[q]);
        const uint32_t n = mine ? min(static_cast<uint32_t>(a.ccnt[i]), a.B) : 0u;
        uint32_t quota = 0, pos = 0, pos2 = 0;
        if (n) {
            quota = a.quota[i];
            pos = a.base[i];
            pos2 = a.base2[i];
            atomicMin(&run_lo[0], pos);
            atomicMin(&run_lo[1], pos2);
        }
        __syncthreads();
        const uint32_t lo = run_lo[0], lo2 = run_lo[1];
        uint32_t* out = a.cands + q * a.m;
        const uint4* buf = reinterpret_cast<const uint4*>(cb_base(a, q, p < a.P ? p : 0u));
        uint32_t at = pos - lo, at2 = pos2 - lo2;  // staging offsets of this thread's next kept ids
        for (uint32_t e0 = 0; e0 < n; e0 += 64) {
            uint4 v[8];
#pragma unroll
            for (uint32_t u = 0; u < 8; ++u) v[u] = e0 + 8 * u < n ? __ldcs(buf + (e0 >> 3) + u) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
            for (uint32_t u = 0; u < 8; ++u) {
                if (e0 + 8 * u >= n) break;  // (pieces past the tie cut hold a few entries: one or two words)
                const uint32_t w4[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                for (uint32_t h = 0; h < 8; ++h) {
                    const uint32_t x = (w4[h >> 1] >> (16 * (h & 1u))) & 0xffffu;
                    const bool valid = e0 + 8 * u + h < n;
                    const bool gt = (x & 0x8000u) != 0;
                    const bool tie = valid && !gt && quota != 0;  // the first ties in id order
                    const uint32_t id = pbase + (x & 0x7fffu);
                    if (valid && gt) {
                        if (at < kCompactStage) stage[0][at] = id;
                        else __stcs(out + lo + at, id);
                        ++at;
                    } else if (tie) {
                        if (at2 < kCompactStage) stage[1][at2] = id;
                        else __stcs(out + lo2 + at2, id);
                        ++at2;
                    }
                    quota -= tie ? 1u : 0u;
                }
            }
        }
        if (n) {
            atomicMax(&run_hi[0], at);
            atomicMax(&run_hi[1], at2);
        }
        __syncthreads();
        const uint32_t len = min(run_hi[0], kCompactStage), len2 = min(run_hi[1], kCompactStage);
        for (uint32_t t = threadIdx.x; t < len; t += blockDim.x) __stcs(out + lo + t, stage[0][t]);
        for (uint32_t t = threadIdx.x; t < len2; t += blockDim.x) __stcs(out + lo2 + t, stage[1][t]);
        __syncthreads();  // the staging areas and run bounds are reused by the next query
    }
}

// K4 (default): a warp per (query, piece). A lane reads four consecutive entries (8 bytes; the warp
// 128 entries = 256 contiguous bytes per load), keeps every score > T entry and the first `quota`
// ties (id order = buffer order = (lane, h) order), and writes consecutive output positions.
__device__ __forceinline__ void st_cs_if(bool p, uint32_t* addr, uint32_t v) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %0, 0;\n\t@q st.global.cs.u32 [%1], %2;\n\t}"
                 :
                 : "r"(static_cast<uint32_t>(p)), "l"(addr), "r"(v)
                 : "memory");
}

__device__ __forceinline__ uint2 cb_load4(const DenseArgs& a, const uint16_t* buf, uint32_t e, uint32_t n) {
    uint2 v = make_uint2(0u, 0u);
    if (e < n) {
        if ((a.B & 3u) == 0) {  // buffers start 8-byte aligned and e + 3 < B
            v = __ldcs(reinterpret_cast<const uint2*>(buf + e));
        } else {
            const uint32_t x0 = __ldcs(buf + e), x1 = e + 1 < n ? __ldcs(buf + e + 1) : 0u;
            const uint32_t x2 = e + 2 < n ? __ldcs(buf + e + 2) : 0u, x3 = e + 3 < n ? __ldcs(buf + e + 3) : 0u;
            v = make_uint2(x0 | (x1 << 16), x2 | (x3 << 16));
        }
    }
    return v;
}

__global__ void __launch_bounds__(256, 5) dense_compact_kernel(DenseArgs a) {
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint32_t p = blockIdx.x * 8 + warp;
    if (p >= a.P) return;
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t pbase = p * a.WP;
    const uint32_t nlist = a.nclist[0];
    // The next work item's counts, quota, offsets and first 128 entries are loaded while this one
    // is processed (the loop is latency-bound otherwise: one dependent round trip per item).
    struct Item {
        uint64_t q;
        uint32_t n, quota, pos, pos2;
        uint2 x;
    };
    const uint32_t gp = gpiece(a, p);
    auto fetch = [&](uint32_t j, Item& it) {
        it.q = a.clist[j];  // an unflagged query with a dense superset
        const uint64_t i = it.q * a.P + p;
        const uint16_t* buf = cb_base(a, it.q, p);
        // pieces past the query's tie cut hold a few score > T entries: the thread kernel's (by
        // superset density); everything else loads at once: counts, quota, offsets, 128 entries
        const bool mine = a.compact_mode != 0 || !a.pcut || gp < a.pcut[it.q];
        it.n = 0;
        it.quota = it.pos = it.pos2 = 0;
        it.x = make_uint2(0u, 0u);
        if (mine) {
            // the entries first, under the buffer's capacity (their count arrives with them)
            it.x = cb_load4(a, buf, 4 * lane, a.B);
            it.n = min(static_cast<uint32_t>(a.ccnt[i]), a.B);
            it.quota = a.quota[i];
            it.pos = a.base[i];    // score > T entries
            it.pos2 = a.base2[i];  // ties
        }
    };
    Item cur;
    if (blockIdx.y < nlist) fetch(blockIdx.y, cur);
    for (uint32_t j = blockIdx.y; j < nlist; j += gridDim.y) {
        Item nxt;
        if (j + gridDim.y < nlist) fetch(j + gridDim.y, nxt);
        const uint32_t n = cur.n, quota = cur.quota;
        uint32_t pos = cur.pos, pos2 = cur.pos2, ties = 0;
        uint32_t* out = a.cands + cur.q * a.m;
        const uint16_t* buf = cb_base(a, cur.q, p);
        for (uint32_t e0 = 0; e0 < n; e0 += 128) {
            const uint32_t e = e0 + 4 * lane;
            const uint2 v = e0 == 0 ? cur.x : cb_load4(a, buf, e, n);
            // this lane's four entries as 4-bit masks: score > T, ties (valid entries only)
            const uint32_t nv = e < n ? min(n - e, 4u) : 0u;
            const uint32_t vmask = (1u << nv) - 1u;
            const uint32_t gbits = ((v.x >> 15) & 1u) | ((v.x >> 30) & 2u) | ((v.y >> 13) & 4u) | ((v.y >> 28) & 8u);
            const uint32_t gm = gbits & vmask, tm = ~gbits & vmask;
            // entries before this lane's in id order: one inclusive warp scan of both counts
            const uint32_t own = __popc(gm) | (__popc(tm) << 16);
            uint32_t inc = own;
#pragma unroll
            for (uint32_t d = 1; d < 32; d <<= 1) {
                const uint32_t up = __shfl_up_sync(kFull, inc, d);
                if (lane >= d) inc += up;
            }
            const uint32_t tot = __shfl_sync(kFull, inc, 31);
            const uint32_t before = inc - own;
            uint32_t gpos = pos + (before & 0xffffu);
            uint32_t tbefore = before >> 16;
            const uint32_t room = quota > ties ? quota - ties : 0u;  // ties of this step still kept
            const uint32_t xs[4] = {v.x & 0x7fffu, (v.x >> 16) & 0x7fffu, v.y & 0x7fffu, (v.y >> 16) & 0x7fffu};
#pragma unroll
            for (uint32_t h = 0; h < 4; ++h) {
                const bool g = (gm >> h) & 1u, t = (tm >> h) & 1u;
                st_cs_if(g, out + gpos, pbase + xs[h]);  // predicated stores: no branch per entry
                st_cs_if(t && tbefore < room, out + pos2 + tbefore, pbase + xs[h]);
                gpos += g ? 1u : 0u;
                tbefore += t ? 1u : 0u;
            }
            pos += tot & 0xffffu;
            pos2 += min(tot >> 16, room);
            ties += tot >> 16;
        }
        cur = nxt;
    }
}

__global__ void dense_flag_list_kernel(DenseArgs a) {  // qmap <- flagged queries (any order)
    const uint64_t q = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (q < a.nq && a.qflag[q]) a.qmap[atomicAdd(a.nmap, 1u)] = static_cast<uint32_t>(q);
}

__global__ void dense_codes_fill_kernel(uint16_t* codes, uint64_t count, uint16_t none) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count; i += uint64_t(gridDim.x) * blockDim.x)
        codes[i] = none;
}

__global__ void dense_codes_kernel(const uint32_t* ids, const uint32_t* cell_off, uint64_t n, uint32_t ns, uint32_t K,
                                   uint16_t* codes, uint32_t cw) {  // cw = codes per point (8 or 16)
    const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (t >= uint64_t(ns) * K) return;
    const uint32_t s = static_cast<uint32_t>(t / K), cell = static_cast<uint32_t>(t % K);
    const uint32_t* off = cell_off + uint64_t(s) * (K + 1);
    const uint32_t* sid = ids + uint64_t(s) * n;
    const uint16_t code = static_cast<uint16_t>(dense_slot(ns, K, s, cell));
    // grouped layout: point p keeps subspace s at position (s - p) % 8 (lane-rotated lookups)
    if (dense_grouped(ns)) {
        for (uint32_t i = off[cell]; i < off[cell + 1]; ++i) codes[uint64_t(sid[i]) * cw + ((s - sid[i]) & 7u)] = code;
    } else {
        for (uint32_t i = off[cell]; i < off[cell + 1]; ++i) codes[uint64_t(sid[i]) * cw + s] = code;
    }
}

// Bank-conflict schedule of a 32-point tile's lookups (grouped layout). Lookup j of the fused
// pass reads code position j of every lane's point, and a code is its whole slot (s*K + cell in
// the grouped form), so a point's 8 codes may sit in any order: the carry-save sum does not care.
// A warp-wide lookup costs as many shared wavefronts as the most-loaded bank (slot & 31) among the
// 32 lanes' slots; with the lane-rotated start (lane l reads subspace (j + l) % 8 at step j), four
// lanes share each subspace's four banks at random: 2.95 wavefronts per lookup at cfg4. Here one
// thread per tile reorders each point's codes by local search: swapping two positions of one
// point moves one slot between two steps, accepted when the steps' cost (max bank load, then the
// number of banks at that max) drops. (Two lanes reading the very same slot broadcast; the model
// counts them twice, which only errs on the safe side.) One pass takes random tiles from 2.96 to
// about 2.0 wavefronts per lookup in a simulation (the max-bank-degree bound is 1.67).
// The half-width interleaved codes (v = c' * 4 + s / 2, bank v % 32) take the same search with
// swaps restricted to positions of equal parity (HALF).
template <bool HALF>
__global__ void __launch_bounds__(64) dense_codes_sched_kernel(uint16_t* codes, uint64_t ntiles, uint32_t passes) {
    const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (t >= ntiles) return;
    uint4* row = reinterpret_cast<uint4*>(codes) + t * 32;
    uint32_t c[32][4];  // the tile's codes, two per word (position 2i in the low half)
    uint8_t load[8][32], hist[8][33], mx[8];
    for (uint32_t j = 0; j < 8; ++j) {
        for (uint32_t b = 0; b < 32; ++b) load[j][b] = 0;
        for (uint32_t v = 0; v < 33; ++v) hist[j][v] = 0;
    }
    auto code = [&](uint32_t l, uint32_t j) -> uint32_t { return (c[l][j >> 1] >> (16 * (j & 1u))) & 0xffffu; };
    for (uint32_t l = 0; l < 32; ++l) {
        const uint4 v = row[l];
        c[l][0] = v.x, c[l][1] = v.y, c[l][2] = v.z, c[l][3] = v.w;
        for (uint32_t j = 0; j < 8; ++j) ++load[j][code(l, j) & 31u];
    }
    for (uint32_t j = 0; j < 8; ++j) {
        mx[j] = 0;
        for (uint32_t b = 0; b < 32; ++b) {
            ++hist[j][load[j][b]];
            mx[j] = max(mx[j], load[j][b]);
        }
    }
    auto inc = [&](uint32_t j, uint32_t b) {
        const uint32_t v = load[j][b]++;
        --hist[j][v], ++hist[j][v + 1];
        if (v + 1 > mx[j]) mx[j] = static_cast<uint8_t>(v + 1);
    };
    auto dec = [&](uint32_t j, uint32_t b) {
        const uint32_t v = load[j][b]--;
        --hist[j][v], ++hist[j][v - 1];
        if (v == mx[j] && hist[j][v] == 0) mx[j] = static_cast<uint8_t>(v - 1);
    };
    auto cost = [&](uint32_t j) -> uint32_t { return mx[j] * 64u + hist[j][mx[j]]; };
    for (uint32_t pass = 0; pass < passes; ++pass) {
        for (uint32_t l = 0; l < 32; ++l) {
            for (uint32_t j1 = 0; j1 < 7; ++j1) {
                for (uint32_t j2 = j1 + (HALF ? 2 : 1); j2 < 8; j2 += HALF ? 2 : 1) {
                    const uint32_t b1 = code(l, j1) & 31u, b2 = code(l, j2) & 31u;
                    if (b1 == b2) continue;
                    const uint32_t before = cost(j1) + cost(j2);
                    dec(j1, b1), inc(j1, b2), dec(j2, b2), inc(j2, b1);
                    if (cost(j1) + cost(j2) < before) {
                        const uint32_t x1 = code(l, j1), x2 = code(l, j2);
                        const uint32_t s1 = 16 * (j1 & 1u), s2 = 16 * (j2 & 1u);
                        c[l][j1 >> 1] = (c[l][j1 >> 1] & ~(0xffffu << s1)) | (x2 << s1);
                        c[l][j2 >> 1] = (c[l][j2 >> 1] & ~(0xffffu << s2)) | (x1 << s2);
                    } else {
                        dec(j1, b2), inc(j1, b1), dec(j2, b1), inc(j2, b2);
                    }
                }
            }
        }
    }
    for (uint32_t l = 0; l < 32; ++l) row[l] = make_uint4(c[l][0], c[l][1], c[l][2], c[l][3]);
}

// ------------------------------------------------------------ half-width mode
// For mask tables beyond shared memory at 32 bits per slot (config 5: 8 x 10,000 cells): a CTA
// owns 16 queries and keeps one u16 mask per (subspace, cell). Region s of the table holds K + 1
// slots at s * (K + 1); slot 0 of a region is always zero and a point's code in subspace s is
// cell + 1 (0 for s >= N_s and for the padding rows past n). A lane looks up TWO points of a
// 64-point tile, A = t0 + lane (bits 0-15) and B = t0 + 32 + lane (bits 16-31), so the carry-save
// adders and the 32x32 transpose work on full 32-bit words exactly as in the 32-query kernels.
// After the transpose lane c holds query c & 15 over the 32 points t0 + 32 * (c >> 4) + r.
template <uint32_t kDT>
__device__ void build_masks_h(const DenseArgs& a, uint32_t* M, uint64_t q0, uint32_t nqb) {
    constexpr uint32_t kDW = kDT / 32;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t R = a.K + 1;
    const uint32_t words = (a.ns * R + 1) / 2;
    for (uint32_t i = tid; i < words; i += kDT) M[i] = 0;
    __syncthreads();
    for (uint32_t j = warp; j < nqb; j += kDW) {
        const uint64_t q = a.qmap ? a.qmap[q0 + j] : q0 + j;
        for (uint32_t s = 0; s < a.ns; ++s) {
            const uint64_t t = q * a.ns + s;
            const uint32_t cnt = a.cells_off ? static_cast<uint32_t>(a.cells_off[t + 1] - a.cells_off[t]) : a.ncells[t];
            const uint32_t* cp = a.cells + (a.cells_off ? a.cells_off[t] : t * a.cells_cap);
            for (uint32_t i = lane; i < cnt; i += 32) {
                const uint32_t slot = a.hgroup ? ((cp[i] + 1) << 3) | s : s * R + cp[i] + 1;
                atomicOr(M + (slot >> 1), 1u << (j + ((slot & 1u) << 4)));
            }
        }
    }
    __syncthreads();
}

// Slot of code c' (cell + 1) at code position j. Region layout: s * (K + 1) + c' (positions >= N_s
// read region 0's zero slot). Interleaved layout (eight subspaces, a.hgroup; HG): slot c' * 8 + s,
// so subspaces 2g and 2g + 1 share 32-bit words and the word's bank is (4 c' + g) % 32. The code is
// v = c' * 4 + s / 2 and position j holds a subspace of parity j % 2, so the lookup's byte address
// is 4 v + 2 (j % 2): the odd positions' +2 sits in the load's immediate, and the address is one
// extraction plus one shift-add of the code. Position j of point p holds subspace (j + 2p) % 8 to
// start with, then the codes are reordered against bank conflicts (the bank of a lookup is v % 32;
// dense_codes_sched_kernel swaps positions of equal parity only).
struct RegionOff {
    uint32_t o[8], mb;
    __device__ RegionOff(const DenseArgs& a, const uint32_t* M) {
        mb = static_cast<uint32_t>(__cvta_generic_to_shared(M));
#pragma unroll
        for (uint32_t j = 0; j < 8; ++j) o[j] = j < a.ns ? j * (a.K + 1) : 0u;
    }
};

template <uint32_t IMM>
__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u16 %0, [%1+%2];" : "=r"(v) : "r"(addr), "n"(IMM));
    return v;
}

template <bool HG>
__device__ __forceinline__ void masks_h(const uint16_t* M16, const RegionOff& ro, uint4 ca, uint4 cb, uint32_t (&m)[8]) {
    const uint32_t xa[4] = {ca.x, ca.y, ca.z, ca.w}, xb[4] = {cb.x, cb.y, cb.z, cb.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if constexpr (HG) {
            m[2 * i] = __byte_perm(lds_u16<0>(ro.mb + ((xa[i] & 0xffffu) << 2)),
                                   lds_u16<0>(ro.mb + ((xb[i] & 0xffffu) << 2)), 0x5410);
            m[2 * i + 1] = __byte_perm(lds_u16<2>(ro.mb + ((xa[i] >> 16) << 2)),
                                       lds_u16<2>(ro.mb + ((xb[i] >> 16) << 2)), 0x5410);
        } else {
            m[2 * i] = uint32_t(M16[ro.o[2 * i] + (xa[i] & 0xffffu)]) |
                       (uint32_t(M16[ro.o[2 * i] + (xb[i] & 0xffffu)]) << 16);
            m[2 * i + 1] = uint32_t(M16[ro.o[2 * i + 1] + (xa[i] >> 16)]) |
                           (uint32_t(M16[ro.o[2 * i + 1] + (xb[i] >> 16)]) << 16);
        }
    }
}

__device__ __forceinline__ void csa_h(const uint32_t (&m)[8], uint32_t (&b)[4]) {
    uint32_t s1, c1, s2, c2, b0, c4, s5, c5;
    fadd(m[0], m[1], m[2], s1, c1);
    fadd(m[3], m[4], m[5], s2, c2);
    const uint32_t s3 = m[6] ^ m[7], c3 = m[6] & m[7];
    fadd(s1, s2, s3, b0, c4);
    fadd(c1, c2, c3, s5, c5);
    const uint32_t c6 = s5 & c4;
    b[0] = b0;
    b[1] = s5 ^ c4;
    b[2] = c5 ^ c6;
    b[3] = c5 & c6;
}

template <bool HG>
__device__ __forceinline__ void planes_h(const uint16_t* M16, const RegionOff& ro, uint4 ca, uint4 cb,
                                         uint32_t (&b)[4]) {
    uint32_t m[8];
    masks_h<HG>(M16, ro, ca, cb, m);
    csa_h(m, b);
}

// K1 (half width): per (query, piece) #points with score >= t, t = 1..8.
template <uint32_t kDT, bool HG>
__global__ void __launch_bounds__(kDT, 1024 / kDT) dense_hist_h_kernel(DenseArgs a) {
    constexpr uint32_t kDW = kDT / 32;
    extern __shared__ uint32_t M[];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint64_t q0 = uint64_t(blockIdx.x) * 16;
    const uint64_t nvalid = a.qmap ? *a.nmap : a.nq;
    if (q0 >= nvalid) return;
    const uint32_t nqb = static_cast<uint32_t>(min_u64(16, nvalid - q0));
    build_masks_h<kDT>(a, M, q0, nqb);
    const uint32_t row = blockIdx.y * kDW + warp;
    if (row >= a.P) return;
    const uint64_t lo = uint64_t(row) * (a.pstride ? a.pstride : 1u) * a.WP;
    if (lo >= a.n) return;
    const uint64_t hi = min_u64(a.n, lo + a.WP);  // rows past n are zero-code padding: score 0
    const uint16_t* M16 = reinterpret_cast<const uint16_t*>(M);
    const RegionOff ro(a, M);
    const Xpose xp(lane);
    uint32_t cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (uint64_t t0 = lo; t0 < hi; t0 += 64) {
        uint32_t b[4];
        planes_h<HG>(M16, ro, __ldg(a.codes + t0 + lane), __ldg(a.codes + t0 + 32 + lane), b);
        const uint32_t B0 = xp(b[0]), B1 = xp(b[1]), B2 = xp(b[2]), B3 = xp(b[3]);
        const uint32_t g8 = B3, g4 = B3 | B2, g2 = g4 | B1, g1 = g2 | B0;
        const uint32_t g6 = B3 | (B2 & B1), g5 = B3 | (B2 & (B1 | B0)), g7 = B3 | (B2 & B1 & B0);
        const uint32_t g3 = g4 | (B1 & B0);
        cnt[0] += __popc(g1);
        cnt[1] += __popc(g2);
        cnt[2] += __popc(g3);
        cnt[3] += __popc(g4);
        cnt[4] += __popc(g5);
        cnt[5] += __popc(g6);
        cnt[6] += __popc(g7);
        cnt[7] += __popc(g8);
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) cnt[t] += __shfl_xor_sync(kFull, cnt[t], 16);  // the tile's two halves
    if (lane < nqb) {
        uint4 v;
        v.x = cnt[0] | (cnt[1] << 16);
        v.y = cnt[2] | (cnt[3] << 16);
        v.z = cnt[4] | (cnt[5] << 16);
        v.w = cnt[6] | (cnt[7] << 16);
        const uint64_t q = a.qmap ? a.qmap[q0 + lane] : q0 + lane;
        reinterpret_cast<uint4*>(a.hist)[q * a.P + row] = v;
    }
}

// K3 (half width): lanes c and c + 16 share query c; ties and output slots are taken in id order
// (the first half of a tile before the second).
template <uint32_t kDT, bool HG>
__global__ void __launch_bounds__(kDT, 1024 / kDT) dense_emit_h_kernel(DenseArgs a) {
    constexpr uint32_t kDW = kDT / 32;
    extern __shared__ uint32_t M[];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint64_t q0 = uint64_t(blockIdx.x) * 16;
    const uint64_t nvalid = a.qmap ? *a.nmap : a.nq;
    if (q0 >= nvalid) return;
    const uint32_t nqb = static_cast<uint32_t>(min_u64(16, nvalid - q0));
    build_masks_h<kDT>(a, M, q0, nqb);
    const uint32_t piece = blockIdx.y * kDW + warp;
    if (piece >= a.P) return;
    const uint64_t lo = uint64_t(piece) * a.WP;
    const uint64_t hi = min_u64(a.n, lo + a.WP);
    const uint32_t qj = lane & 15u, half = lane >> 4;
    const bool mine = qj < nqb;
    const uint64_t q = !mine ? 0 : a.qmap ? a.qmap[q0 + qj] : q0 + qj;
    const uint32_t T = mine ? a.T[q] : 0u;
    const uint32_t quota = mine ? a.quota[q * a.P + piece] : 0u;
    uint32_t pos = mine ? a.base[q * a.P + piece] : 0u, tseen = 0;
    uint32_t* out = a.cands + q * a.m;
    const uint16_t* M16 = reinterpret_cast<const uint16_t*>(M);
    const RegionOff ro(a, M);
    const Xpose xp(lane);
    for (uint64_t t0 = lo; t0 < hi; t0 += 64) {
        uint32_t b[4];
        planes_h<HG>(M16, ro, __ldg(a.codes + t0 + lane), __ldg(a.codes + t0 + 32 + lane), b);
        const uint32_t B0 = xp(b[0]), B1 = xp(b[1]), B2 = xp(b[2]), B3 = xp(b[3]);
        const uint64_t pb = t0 + 32 * half;  // this lane's first point
        const uint32_t vmask = !mine || pb >= hi ? 0u : hi - pb >= 32 ? kFull : ((1u << (hi - pb)) - 1u);
        const uint32_t Bh[4] = {B0, B1, B2, B3};
        if (a.scores_dbg && q0 == 0 && qj == 0 && mine) {  // parity dump: query 0's scores
            for (uint32_t r = 0; r < 32 && pb + r < hi; ++r) {
                const uint32_t sc = ((B0 >> r) & 1u) | (((B1 >> r) & 1u) << 1) | (((B2 >> r) & 1u) << 2) |
                                    (((B3 >> r) & 1u) << 3);
                a.scores_dbg[pb + r] = static_cast<uint8_t>(sc);
            }
        }
        const uint32_t geT = ge_mask_n<4>(Bh, T) & vmask;
        const uint32_t gt = ge_mask_n<4>(Bh, T + 1) & vmask;
        const uint32_t eq = geT & ~gt;
        const uint32_t ec = __popc(eq), eo = __shfl_xor_sync(kFull, ec, 16);
        const uint32_t seen = tseen + (half ? eo : 0u);  // ties before this lane's points
        uint32_t take = gt;
        if (eq && seen < quota) {
            const uint32_t r = quota - seen;
            uint32_t rest = eq;
            for (uint32_t i = 0; i < r && rest; ++i) rest &= rest - 1;
            take |= eq ^ rest;
        }
        tseen += ec + eo;
        const uint32_t tc = __popc(take), to = __shfl_xor_sync(kFull, tc, 16);
        uint32_t p = pos + (half ? to : 0u);
        while (take) {
            const uint32_t bit = __ffs(take) - 1;
            take &= take - 1;
            __stcs(out + p++, static_cast<uint32_t>(pb) + bit);
        }
        pos += tc + to;
    }
}

// K3' (half width): histograms + per-(query, piece) supersets in one pass (as fused_pieces, 2-byte
// stores; lanes c and c + 16 append to query c's buffer in id order).
template <uint32_t kDT, bool HG>
__global__ void __launch_bounds__(kDT, 1024 / kDT) dense_fused_h_kernel(DenseArgs a) {
    constexpr uint32_t kDW = kDT / 32;
    extern __shared__ uint32_t M[];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint64_t q0 = uint64_t(blockIdx.x) * 16;
    const uint32_t nqb = static_cast<uint32_t>(min_u64(16, a.nq - q0));
    const uint32_t myL = threadIdx.x < nqb ? a.L[q0 + threadIdx.x] : 0u;
    if (!__syncthreads_or((myL & 0xffu) != 0)) return;  // all two-pass
    build_masks_h<kDT>(a, M, q0, nqb);
    const uint32_t qj = lane & 15u, half = lane >> 4;
    const bool mine = qj < nqb;
    // bits j and 16 + j of each word = query j's L bits (the ballot of lanes j and j + 16)
    const uint32_t L = mine ? a.L[q0 + qj] & 0xffu : 0u;
    const uint32_t T0 = __ballot_sync(kFull, L & 1u), T1 = __ballot_sync(kFull, L & 2u);
    const uint32_t T2 = __ballot_sync(kFull, L & 4u), T3 = __ballot_sync(kFull, L & 8u);
    const uint32_t live = __ballot_sync(kFull, L != 0);
    const uint32_t cut = a.pcut && mine ? a.pcut[q0 + qj] : a.P;
    const uint16_t* M16 = reinterpret_cast<const uint16_t*>(M);
    const RegionOff ro(a, M);
    const Xpose xp(lane);
    for (uint32_t k = 0; k < a.ppw; ++k) {
        const uint32_t piece = (blockIdx.y * kDW + warp) * a.ppw + k;
        if (piece >= a.P) return;
        const uint64_t lo = uint64_t(piece) * a.WP;
        const uint64_t hi = min_u64(a.n, lo + a.WP);
        uint32_t cnt = 0, nb = 0;
        uint16_t* buf = cb_base(a, mine ? q0 + qj : q0, piece);
        // 32-bit tile loop (the padded code rows cover a whole last piece and one tile past it);
        // the next tile's mask lookups are in flight while this tile is compared and emitted
        const uint32_t len = static_cast<uint32_t>(hi - lo);
        const uint4* cptr = a.codes + lo + lane;
        uint32_t mk[8];
        masks_h<HG>(M16, ro, __ldg(cptr), __ldg(cptr + 32), mk);
        uint4 ca = __ldg(cptr + 64), cb = __ldg(cptr + 96);
        // past every lane's tie cut only score > L is kept: one transpose per tile (the piece's
        // #(score >= L) is recorded as #(score > L), as in fused_pieces)
        const uint32_t gp = gpiece(a, piece);
        const bool need_ge = __any_sync(kFull, gp < cut);
        // the tile loop, compiled once per piece kind (some query still needs ties / past every tie cut)
        auto tile_loop = [&](auto need_ge_c) {
            constexpr bool NEED_GE = decltype(need_ge_c)::value;
            for (uint32_t tb0 = 0; tb0 < len; tb0 += 64) {
                cptr += 64;
                const uint4 na = __ldg(cptr + 64), nbv = __ldg(cptr + 96);
                uint32_t b[4];
                csa_h(mk, b);
                masks_h<HG>(M16, ro, ca, cb, mk);
                ca = na;
                cb = nbv;
                uint32_t gt = b[3] & ~T3, eq = ~(b[3] ^ T3);
                gt |= eq & b[2] & ~T2;
                eq &= ~(b[2] ^ T2);
                gt |= eq & b[1] & ~T1;
                eq &= ~(b[1] ^ T1);
                gt |= eq & b[0] & ~T0;
                eq &= ~(b[0] ^ T0);
                // queries past the block's last have no live bits: their lanes see empty words
                if constexpr (!NEED_GE) {
                    // past every tie cut: no transpose (fused_pieces); lane p's word holds point t0 + p's
                    // queries in bits 0-15 and point t0 + 32 + p's in bits 16-31, so the A points go
                    // first (id order), each appended by its query's lane of half 0, then the B points by
                    // half 1; both lanes of a query keep its count
                    const uint32_t gl = gt & live;
                    uint32_t pend = __ballot_sync(kFull, gl != 0);
    #pragma unroll
                    for (uint32_t hh = 0; hh < 2; ++hh) {
                        uint32_t pp = pend;
                        while (pp) {
                            const uint32_t p = __ffs(pp) - 1;
                            pp &= pp - 1;
                            const uint32_t hit = (__shfl_sync(kFull, gl, p) >> (16 * hh + qj)) & 1u;  // branch-free
                            const uint32_t own = half == hh ? hit : 0u;
                            if (own && nb < a.B) buf[cb_off(a, nb)] = static_cast<uint16_t>((tb0 + 32 * hh + p) | 0x8000u);
                            cnt += own * 0x10001u;
                            nb += hit;
                        }
                    }
                    continue;
                }
                const uint32_t g1 = xp(gt & live);
                uint32_t kept = g1;
                {
                    const uint32_t ge0 = xp((gt | eq) & live);
                    cnt += __popc(ge0) | (__popc(g1) << 16);
                    if (gp < cut) kept = ge0;  // before the tie cut: every score >= L
                }
                const uint32_t c0 = __popc(kept), o0 = __shfl_xor_sync(kFull, c0, 16);
                uint32_t at = nb + (half ? o0 : 0u);
                const uint32_t tb = tb0 + 32 * half;
                uint32_t bits = kept;
                while (bits) {  // id order
                    const uint32_t r = __ffs(bits) - 1;
                    bits &= bits - 1;
                    if (at < a.B) buf[cb_off(a, at)] = static_cast<uint16_t>((tb + r) | (((g1 >> r) & 1u) << 15));
                    ++at;
                }
                nb += c0 + o0;
            }
        };
        if (need_ge) tile_loop(std::true_type{});
        else tile_loop(std::false_type{});
        cnt += __shfl_xor_sync(kFull, cnt, 16);  // packed 16-bit halves, each <= WP
        if (half == 0 && mine) {
            const uint64_t i = (q0 + qj) * a.P + piece;
            a.h2[i] = cnt;
            a.ccnt[i] = static_cast<uint16_t>(nb);
        }
    }
}

// ----------------------------------------------------- cluster-pair fused pass
// Config 5's tables (8 x 10,000 cells) in a 2-CTA cluster instead of the half-width mode: CTA r of
// the pair keeps 32-bit masks (32 queries) for subspaces 4r .. 4r+3 only (4 x 10,001 slots,
// 160 KB), so one shared-memory lookup serves 32 queries instead of 16 — half the lookups (and
// their bank conflicts) per point and query. A warp of each CTA walks the same piece pairs
// (2p, 2p+1); CTA r finalises piece 2p + r. Per 32-point tile it computes its 3-bit partial scores
// (its four subspaces: 0..4, bit-sliced, lane = point, bit = query) of both pieces' tiles, sends the
// partial of the peer's tile into the peer's ring slot with st.async (completing the peer's
// mbarrier transaction), and adds the peer's partial of its own tile to its own: the 4-bit
// scores of the 32 queries, from which the single pass proceeds exactly as in fused_pieces
// (comparison with L before the transpose, counts, id-ordered buffer entries). The ring runs
// kPairRing - 1 tiles ahead; a consumed slot is released to the producer with a remote
// mbarrier arrive. Uses the half-width mode's point codes (cell + 1 per subspace, 0 = none).
constexpr uint32_t kPairRing = 3;

__device__ __forceinline__ uint32_t cta_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t map_peer(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void pbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void pbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void pbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok) {
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n"
            "}\n"
            : "=r"(ok)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
    }
}
// relaxed: the slot's values are already consumed (data dependence) when the consumer releases it
__device__ __forceinline__ void pbar_arrive_remote(uint32_t remote_bar) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote_bar) : "memory");
}
__device__ __forceinline__ void st_async_v4(uint32_t remote_addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d,
                                            uint32_t remote_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                     remote_addr),
                 "r"(a), "r"(b), "r"(c), "r"(d), "r"(remote_bar)
                 : "memory");
}

// 3-bit partial score planes of 32 points (lane) x 32 queries (bit) over a CTA's four subspaces
__device__ __forceinline__ void pair_partial(const uint32_t* M, uint32_t R, uint2 c, uint32_t (&p)[3]) {
    const uint32_t m0 = M[c.x & 0xffffu], m1 = M[R + (c.x >> 16)];
    const uint32_t m2 = M[2 * R + (c.y & 0xffffu)], m3 = M[3 * R + (c.y >> 16)];
    uint32_t s1, c1;
    fadd(m0, m1, m2, s1, c1);
    p[0] = s1 ^ m3;
    const uint32_t k = s1 & m3;
    p[1] = c1 ^ k;
    p[2] = c1 & k;
}

template <uint32_t kDT>
__global__ void __launch_bounds__(kDT, 1) dense_fused_pair_kernel(DenseArgs a) {
    constexpr uint32_t kDW = kDT / 32;
    extern __shared__ __align__(16) uint32_t M[];
    __shared__ __align__(8) uint64_t full[kDW][kPairRing], empty[kDW][kPairRing];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint32_t r = cta_rank(), peer = r ^ 1u;
    const uint64_t q0 = uint64_t(blockIdx.x >> 1) * 32;
    const uint32_t nqb = static_cast<uint32_t>(min_u64(32, a.nq - q0));
    const uint32_t myL = threadIdx.x < nqb ? a.L[q0 + threadIdx.x] : 0u;
    if (!__syncthreads_or((myL & 0xffu) != 0)) return;  // both CTAs of the pair see the same queries
    const uint32_t R = a.K + 1;
    const uint32_t regions = 4;
    uint4* ring = reinterpret_cast<uint4*>(M + ((regions * R + 3) & ~3u));  // [kDW][kPairRing][32]
    // masks of this CTA's subspaces 4r .. 4r+3 (code = cell + 1; slot 0 of a region stays zero)
    for (uint32_t i = threadIdx.x; i < regions * R; i += kDT) M[i] = 0;
    if (lane < kPairRing) {
        pbar_init(&full[warp][lane], 1);
        pbar_init(&empty[warp][lane], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    for (uint32_t j = warp; j < nqb; j += kDW) {
        const uint64_t q = q0 + j;
        for (uint32_t sl = 0; sl < 4; ++sl) {
            const uint32_t s = 4 * r + sl;
            if (s >= a.ns) break;
            const uint64_t t = q * a.ns + s;
            const uint32_t cnt = a.ncells[t];
            const uint32_t* cp = a.cells + t * a.cells_cap;
            for (uint32_t i = lane; i < cnt; i += 32) atomicOr(M + sl * R + cp[i] + 1, 1u << j);
        }
    }
    __syncthreads();
    cluster_sync_all();  // the peer's barriers are initialised before any remote operation
    // the bits of L[q] across the block's queries: TL[i] bit j = bit i of L[q0 + j]
    const uint32_t L = lane < nqb ? a.L[q0 + lane] & 0xffu : 0u;
    uint32_t TL[4];
#pragma unroll
    for (uint32_t i = 0; i < 4; ++i) TL[i] = __ballot_sync(kFull, (L >> i) & 1u);
    const uint32_t live = __ballot_sync(kFull, L != 0);
    const uint32_t cut = a.pcut && lane < nqb ? a.pcut[q0 + lane] : a.P;
    const Xpose xp(lane);
    uint4* myring = ring + warp * kPairRing * 32;
    const uint32_t peer_ring = map_peer(smem_addr(myring), peer);
    const uint32_t peer_full = map_peer(smem_addr(&full[warp][0]), peer);
    const uint32_t peer_empty = map_peer(smem_addr(&empty[warp][0]), peer);
    const uint2* codes2 = reinterpret_cast<const uint2*>(a.codes);  // 8 u16 codes per point = 2 uint2
    constexpr uint32_t kTiles = kDensePiece / 32, kTileLog = 6;      // tiles per piece (rows padded)
    static_assert(kTiles == (1u << kTileLog), "tiles per piece");
    const uint32_t total = a.ppw * kTiles;                           // the warp's tile sequence
    const uint64_t pair0 = uint64_t(blockIdx.y * kDW + warp) * a.ppw;
    auto piece_of = [&](uint32_t t, uint32_t who) { return (pair0 + (t >> kTileLog)) * 2 + who; };
    auto codes_at = [&](uint32_t t, uint32_t who) -> uint2 {
        const uint64_t pc = piece_of(t, who);
        if (t >= total || pc >= a.P) return make_uint2(0u, 0u);
        return __ldg(codes2 + ((pc << 11) + ((t & (kTiles - 1)) << 5) + lane) * 2 + r);
    };
    // send the partial of tile t of the PEER's piece (codes c) into the peer's ring
    auto send = [&](uint32_t t, uint2 c) {
        const uint32_t slot = t % kPairRing, use = t / kPairRing;
        uint32_t p[3];
        pair_partial(M, R, c, p);
        if (use) pbar_wait(&empty[warp][slot], (use - 1) & 1u);  // the peer has read the slot's last use
        st_async_v4(peer_ring + (slot * 32 + lane) * 16, p[0], p[1], p[2], 0u, peer_full + slot * 8);
    };
    // codes one tile ahead: the next send's (peer piece) and the next own tile's
    uint2 pc_next = codes_at(0, peer);
    for (uint32_t t = 0; t + 1 < kPairRing && t < total; ++t) {
        const uint2 c = pc_next;
        pc_next = codes_at(t + 1, peer);
        send(t, c);
    }
    uint2 own_next = codes_at(0, r);
    uint32_t cnt = 0, nb = 0;
    uint16_t* buf = nullptr;
    for (uint32_t t = 0; t < total; ++t) {
        if (t + kPairRing - 1 < total) {
            const uint2 c = pc_next;
            pc_next = codes_at(t + kPairRing, peer);
            send(t + kPairRing - 1, c);
        }
        const uint32_t j = t & (kTiles - 1);
        const uint64_t piece = piece_of(t, r);
        if (j == 0) {
            cnt = 0;
            nb = 0;
            const uint64_t q = lane < nqb ? q0 + lane : q0;  // idle lanes append nothing
            buf = cb_base(a, q, piece < a.P ? static_cast<uint32_t>(piece) : 0u);
        }
        const uint2 oc = own_next;
        own_next = codes_at(t + 1, r);
        uint32_t own[3];
        pair_partial(M, R, oc, own);
        const uint32_t slot = t % kPairRing;
        if (lane == 0) pbar_expect_tx(&full[warp][slot], 32 * 16);
        pbar_wait(&full[warp][slot], (t / kPairRing) & 1u);
        const uint4 pv = myring[slot * 32 + lane];
        // 4-bit scores = own + peer (3-bit + 3-bit)
        const uint32_t b0 = own[0] ^ pv.x, k0 = own[0] & pv.x;
        const uint32_t t1 = own[1] ^ pv.y, b1 = t1 ^ k0, k1 = (own[1] & pv.y) | (t1 & k0);
        const uint32_t t2 = own[2] ^ pv.z, b2 = t2 ^ k1, k2 = (own[2] & pv.z) | (t2 & k1);
        __syncwarp();  // every lane has consumed its word of the slot
        if (lane == 0) pbar_arrive_remote(peer_empty + slot * 8);  // the slot is free for the peer
        const uint32_t b[4] = {b0, b1, b2, k2};
        uint32_t gt = b[3] & ~TL[3], eq = ~(b[3] ^ TL[3]);
#pragma unroll
        for (int i = 2; i >= 0; --i) {
            gt |= eq & b[i] & ~TL[i];
            eq &= ~(b[i] ^ TL[i]);
        }
        const uint32_t ge0 = xp((gt | eq) & live);  // lane = query, bit = point j * 32 + bit
        const uint32_t g1 = xp(gt & live);
        cnt += __popc(ge0) | (__popc(g1) << 16);
        if (piece < a.P) {
            uint32_t bits = piece < cut ? ge0 : g1;  // past the tie cut: score > L only
            const uint32_t tb = j * 32;
            while (bits) {  // id order
                const uint32_t bit = __ffs(bits) - 1;
                bits &= bits - 1;
                if (nb < a.B) buf[cb_off(a, nb)] = static_cast<uint16_t>((tb + bit) | (((g1 >> bit) & 1u) << 15));
                ++nb;
            }
            if (j + 1 == kTiles && lane < nqb) {
                const uint64_t i = (q0 + lane) * a.P + piece;
                a.h2[i] = cnt;
                a.ccnt[i] = static_cast<uint16_t>(nb);
            }
        }
    }
    cluster_sync_all();  // no CTA leaves while its peer may still write into its ring
}

__global__ void dense_codes_half_kernel(const uint32_t* ids, const uint32_t* cell_off, uint64_t n, uint32_t ns,
                                        uint32_t K, uint16_t* codes, uint32_t group) {
    const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (t >= uint64_t(ns) * K) return;
    const uint32_t s = static_cast<uint32_t>(t / K), cell = static_cast<uint32_t>(t % K);
    const uint32_t* off = cell_off + uint64_t(s) * (K + 1);
    const uint32_t* sid = ids + uint64_t(s) * n;
    // interleaved layout: code (cell + 1) * 4 + s / 2 at a position of s's parity (the lookup adds
    // the position's parity), lane-rotated: position j of point p holds subspace (j + 2p) % 8
    const uint16_t code = static_cast<uint16_t>(group ? ((cell + 1) << 2) | (s >> 1) : cell + 1);
    for (uint32_t i = off[cell]; i < off[cell + 1]; ++i)
        codes[uint64_t(sid[i]) * 8 + (group ? (s - 2 * sid[i]) & 7u : s)] = code;
}

}  // namespace

bool dense_half_supported(uint32_t ns, uint32_t K) {
    return ns >= 1 && ns <= 8 && K + 1 <= 65535 && (uint64_t(ns) * (K + 1) + 1) * 2 <= 200 * 1024;
}

static size_t dense_half_smem(uint32_t ns, uint32_t K) { return ((size_t(ns) * (K + 1) + 1) / 2) * 4; }

cudaError_t launch_dense_codes_half(const uint32_t* ids, const uint32_t* cell_off, uint64_t n, uint64_t n_pad,
                                    uint32_t ns, uint32_t K, uint16_t* codes, uint32_t group, uint32_t sched_passes,
                                    cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(codes, 0, n_pad * 8 * sizeof(uint16_t), st);
    if (e != cudaSuccess) return e;
    const uint64_t total = uint64_t(ns) * K;
    dense_codes_half_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(ids, cell_off, n, ns, K, codes,
                                                                                       group);
    if (group && sched_passes) {
        const uint64_t ntiles = (n + 31) / 32;
        dense_codes_sched_kernel<true><<<static_cast<unsigned>((ntiles + 63) / 64), 64, 0, st>>>(codes, ntiles, sched_passes);
    }
    return cudaGetLastError();
}

template <uint32_t kDT, int KIND>  // 0 hist, 1 emit, 2 fused
static cudaError_t launch_h_t(const DenseArgs& a, size_t smem, cudaStream_t st) {
    auto kern = a.hgroup ? (KIND == 0 ? dense_hist_h_kernel<kDT, true>
                            : KIND == 1 ? dense_emit_h_kernel<kDT, true> : dense_fused_h_kernel<kDT, true>)
                         : (KIND == 0 ? dense_hist_h_kernel<kDT, false>
                            : KIND == 1 ? dense_emit_h_kernel<kDT, false> : dense_fused_h_kernel<kDT, false>);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    constexpr uint32_t kDW = kDT / 32;
    const uint64_t qblocks = (a.nq + 15) / 16;
    DenseArgs b = a;
    uint32_t per_cta = kDW;
    if (KIND == 2) {
        int sms = 148, dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        b.ppw = kFusedPPW;
        if (qblocks * ((a.P + kDW * b.ppw - 1) / (kDW * b.ppw)) < 4ull * sms) b.ppw = 1;
        per_cta = kDW * b.ppw;
    }
    const dim3 grid(static_cast<unsigned>(qblocks), (a.P + per_cta - 1) / per_cta);
    kern<<<grid, kDT, smem, st>>>(b);
    return cudaGetLastError();
}

template <int KIND>
static cudaError_t launch_h(const DenseArgs& a, cudaStream_t st) {
    if (a.nq == 0) return cudaSuccess;
    const size_t smem = dense_half_smem(a.ns, a.K);
    return smem <= 110 * 1024 ? launch_h_t<512, KIND>(a, smem, st) : launch_h_t<1024, KIND>(a, smem, st);
}

bool dense_supported(uint32_t ns, uint32_t K) {
    const uint64_t slots = uint64_t(dense_none(ns, K)) + 1;
    return ns >= 1 && ns <= 8 && slots <= 65535 && slots * 4 <= 200 * 1024;
}

bool dense_wide_supported(uint32_t ns, uint32_t K) {
    return ns >= 9 && ns <= 16 && uint64_t(ns) * K + 1 <= 65535 && (uint64_t(ns) * K + 1) * 4 <= 200 * 1024;
}

size_t dense_smem(uint32_t ns, uint32_t K) { return (size_t(dense_none(ns, K)) + 1) * 4; }

cudaError_t launch_dense_codes(const uint32_t* ids, const uint32_t* cell_off, uint64_t n, uint32_t ns, uint32_t K,
                               uint16_t* codes, uint32_t sched_passes, cudaStream_t st) {
    const uint32_t cw = ns > 8 ? 16 : 8;
    const uint64_t count = (n + kDenseCodePad) * cw;  // the padding rows: zero-slot codes
    const unsigned fb = static_cast<unsigned>(min_u64((count + 255) / 256, 148ull * 16));
    dense_codes_fill_kernel<<<fb ? fb : 1, 256, 0, st>>>(codes, count, static_cast<uint16_t>(dense_none(ns, K)));
    const uint64_t total = uint64_t(ns) * K;
    dense_codes_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(ids, cell_off, n, ns, K, codes, cw);
    if (dense_grouped(ns) && sched_passes) {
        const uint64_t ntiles = (n + 31) / 32;
        dense_codes_sched_kernel<false><<<static_cast<unsigned>((ntiles + 63) / 64), 64, 0, st>>>(codes, ntiles, sched_passes);
    }
    return cudaGetLastError();
}

// 64-query blocks (two mask words per slot) when those masks fit 200 KB: each
// random mask lookup then serves 64 queries; else 32-query blocks.
struct Shape {
    uint32_t threads, words;
    size_t smem;
};
static Shape dense_shape(const DenseArgs& a) {
    const size_t smem1 = dense_smem(a.ns, a.K);
    // the single-pass pipeline measured faster with 32-query blocks (3.75 vs 3.89 ms at cfg2),
    // the two-pass one with 64-query blocks (5.04 vs 5.52 ms)
    const bool allow2 = (a.words ? a.words == 2 : a.cbuf == nullptr) && a.nc != 2;  // 16 subspaces: one word
    if (allow2 && 2 * smem1 <= 200 * 1024) return {1024, 2, 2 * smem1};
    return {smem1 <= 110 * 1024 ? 512u : 1024u, 1, smem1};
}

template <uint32_t kDT, uint32_t W, bool EMIT, uint32_t NC = 1>
static cudaError_t launch_scan(const DenseArgs& a, size_t smem, cudaStream_t st) {
    auto kern = EMIT ? dense_emit_kernel<kDT, W, NC> : dense_hist_kernel<kDT, W, NC>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    constexpr uint32_t kDW = kDT / 32;
    const dim3 grid(static_cast<unsigned>((a.nq + 32 * W - 1) / (32 * W)), (a.P + kDW - 1) / kDW);
    kern<<<grid, kDT, smem, st>>>(a);
    return cudaGetLastError();
}

template <bool EMIT>
static cudaError_t launch_scan_any(const DenseArgs& a, cudaStream_t st) {
    if (a.nq == 0) return cudaSuccess;
    const Shape sh = dense_shape(a);
    if (a.nc == 2) {
        return sh.threads == 512 ? launch_scan<512, 1, EMIT, 2>(a, sh.smem, st)
                                 : launch_scan<1024, 1, EMIT, 2>(a, sh.smem, st);
    }
    if (sh.words == 2) return launch_scan<1024, 2, EMIT>(a, sh.smem, st);
    return sh.threads == 512 ? launch_scan<512, 1, EMIT>(a, sh.smem, st) : launch_scan<1024, 1, EMIT>(a, sh.smem, st);
}

__global__ void dense_rows_kernel(DenseArgs a, uint32_t* out) {  // u16 x 8 -> [len, #>=1..#>=ns, 0] u32
    const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (i >= a.nq * a.P) return;
    const uint32_t p = static_cast<uint32_t>(i % a.P);
    const uint4 v = reinterpret_cast<const uint4*>(a.hist)[i];
    uint32_t* o = out + i * (a.ns + 2);
    o[0] = static_cast<uint32_t>(min_u64(a.WP, a.n - uint64_t(p) * a.WP));
    for (uint32_t t = 1; t <= a.ns; ++t) o[t] = level(v, t);
    o[a.ns + 1] = 0;
}

cudaError_t launch_dense_hist(const DenseArgs& a, cudaStream_t st) {
    return a.half ? launch_h<0>(a, st) : launch_scan_any<false>(a, st);
}
cudaError_t launch_dense_emit(const DenseArgs& a, cudaStream_t st) {
    return a.half ? launch_h<1>(a, st) : launch_scan_any<true>(a, st);
}

cudaError_t launch_dense_hist_rows(const DenseArgs& a, uint32_t* out, cudaStream_t st) {
    const uint64_t total = a.nq * a.P;
    if (total == 0) return cudaSuccess;
    dense_rows_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(a, out);
    return cudaGetLastError();
}

template <uint32_t kDT, uint32_t W, uint32_t NC = 1>
static cudaError_t launch_fused_t(const DenseArgs& a, size_t smem, cudaStream_t st) {
    cudaError_t e = cudaFuncSetAttribute(dense_fused_kernel<kDT, W, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    constexpr uint32_t kDW = kDT / 32;
    // pieces per warp: kFusedPPW amortises the mask build, unless that leaves fewer than about
    // four CTAs per SM in the grid (small batches / corpora: one piece per warp)
    const uint64_t qblocks = (a.nq + 32 * W - 1) / (32 * W);
    int sms = 148, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    DenseArgs b = a;
    b.ppw = std::max<uint32_t>(1u, kFusedPPW * kDensePiece / a.WP);  // about 8192 points per warp
    if (qblocks * ((a.P + kDW * b.ppw - 1) / (kDW * b.ppw)) < 4ull * sms) b.ppw = 1;
    const uint32_t per_cta = kDW * b.ppw;
    const dim3 grid(static_cast<unsigned>(qblocks), (a.P + per_cta - 1) / per_cta);
    dense_fused_kernel<kDT, W, NC><<<grid, kDT, smem, st>>>(b);
    return cudaGetLastError();
}

size_t dense_pair_smem(uint32_t K) {
    return ((size_t(4) * (K + 1) + 3) & ~size_t(3)) * 4 + size_t(32) * kPairRing * 32 * 16;
}

bool dense_pair_supported(uint32_t ns, uint32_t K) {
    return ns >= 5 && ns <= 8 && K + 1 <= 65535 && dense_pair_smem(K) <= 220 * 1024;
}

static cudaError_t launch_fused_pair(const DenseArgs& a, cudaStream_t st) {
    constexpr uint32_t kDT = 1024, kDW = kDT / 32;
    const size_t smem = dense_pair_smem(a.K);
    auto kern = dense_fused_pair_kernel<kDT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    DenseArgs b = a;
    const uint64_t qblocks = (a.nq + 31) / 32;
    const uint64_t pairs = (a.P + 1) / 2;
    int sms = 148, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // piece pairs per warp: kFusedPPW / 2 amortises the mask build unless that starves the grid
    b.ppw = kFusedPPW / 2 ? kFusedPPW / 2 : 1;
    if (2 * qblocks * ((pairs + kDW * b.ppw - 1) / (kDW * b.ppw)) < 4ull * sms) b.ppw = 1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(2 * qblocks), static_cast<unsigned>((pairs + kDW * b.ppw - 1) / (kDW * b.ppw)));
    cfg.blockDim = dim3(kDT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, b);
}

// K0 of the single pass: histograms of every pstride-th short piece.
cudaError_t launch_dense_sample(const DenseArgs& a, cudaStream_t st) {
    DenseArgs s0 = a;
    s0.qmap = nullptr;
    s0.P = a.Ps;
    s0.hist = a.hsample;
    if (a.sWP) s0.WP = a.sWP;  // short sampled pieces: many warps per CTA row, few tiles each
    return launch_dense_hist(s0, st);
}

// K3' of the single pass: the fused histogram + superset pass (kernel by table shape).
cudaError_t launch_dense_fused_pass(const DenseArgs& a, cudaStream_t st) {
    if (a.half && a.pair) return launch_fused_pair(a, st);
    if (a.half) return launch_h<2>(a, st);
    const Shape sh = dense_shape(a);
    if (a.nc == 2) return sh.threads == 512 ? launch_fused_t<512, 1, 2>(a, sh.smem, st) : launch_fused_t<1024, 1, 2>(a, sh.smem, st);
    if (sh.words == 2) return launch_fused_t<1024, 2>(a, sh.smem, st);
    return sh.threads == 512 ? launch_fused_t<512, 1>(a, sh.smem, st) : launch_fused_t<1024, 1>(a, sh.smem, st);
}

// K4 of the single pass: the compaction kernels over the plan's work lists.
cudaError_t launch_dense_compaction(const DenseArgs& a, cudaStream_t st) {
    const unsigned qrows = static_cast<unsigned>(min_u64(a.nq, 1024));  // rows walk the work lists
    if (a.compact_mode != 2) dense_compact_thread_kernel<false><<<dim3((a.P + 255) / 256, qrows), 256, 0, st>>>(a);  // sparse
    if (a.compact_mode == 0 && a.pcut)  // dense supersets past their tie cuts
        dense_compact_thread_kernel<true><<<dim3((a.P + 255) / 256, qrows), 256, 0, st>>>(a);
    if (a.compact_mode != 1) {  // dense supersets: a warp per (query, piece); rows walk the work list
        // (measured at cfg4: 1024 / 4096 / 65535 grid rows -> 29.73 / 29.86 / 30.06 ms per step)
        const unsigned wrows = static_cast<unsigned>(min_u64(a.nq, a.compact_rows ? a.compact_rows : 1024));
        dense_compact_kernel<<<dim3((a.P + 7) / 8, wrows), 256, 0, st>>>(a);
    }
    return cudaGetLastError();
}

cudaError_t launch_dense_select_fused(const DenseArgs& args, cudaStream_t st, cudaEvent_t main_done,
                                      cudaStream_t fb_st) {
    if (args.nq == 0) return cudaSuccess;
    DenseArgs a = args;  // every pass but the fallback emission sees the queries unmapped
    a.qmap = nullptr;
    // K0: histograms of every pstride-th piece, then the speculative bound L per query
    cudaError_t e = launch_dense_sample(a, st);
    if (e != cudaSuccess) return e;
    dense_bound_kernel<<<static_cast<unsigned>((a.nq + 7) / 8), 256, 0, st>>>(a);
    // K3': histograms + supersets in one pass
    e = launch_dense_fused_pass(a, st);
    if (e != cudaSuccess) return e;
    // plan (+ fallback flags and the compaction work lists) from the two levels, compaction
    e = cudaMemsetAsync(a.nclist, 0, 2 * sizeof(uint32_t), st);
    if (e != cudaSuccess) return e;
    dense_plan_fused_kernel<<<static_cast<unsigned>((a.nq + 7) / 8), 256, 0, st>>>(a);
    e = launch_dense_compaction(a, st);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(args.nmap, 0, 4, st);
    if (e != cudaSuccess) return e;
    dense_flag_list_kernel<<<static_cast<unsigned>((a.nq + 255) / 256), 256, 0, st>>>(args);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    // every unflagged query's candidates are final here; the fallback may run on its own stream
    if (main_done) {
        e = cudaEventRecord(main_done, st);
        if (e != cudaSuccess) return e;
        if (fb_st) {
            e = cudaStreamWaitEvent(fb_st, main_done, 0);
            if (e != cudaSuccess) return e;
            st = fb_st;
        }
    }
    // the flagged queries (T != L) get the exact two-pass select — full histograms, plan,
    // emission — through qmap; blocks past the flagged count exit at once
    DenseArgs fb = args;
    fb.qflag = nullptr;
    fb.pstride = 1;
    e = launch_dense_hist(fb, st);
    if (e != cudaSuccess) return e;
    dense_plan_kernel<<<static_cast<unsigned>((a.nq + 7) / 8), 256, 0, st>>>(fb);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_dense_emit(fb, st);
}

cudaError_t launch_dense_select(const DenseArgs& a, cudaStream_t st) {
    if (a.nq == 0) return cudaSuccess;
    cudaError_t e = launch_dense_hist(a, st);
    if (e != cudaSuccess) return e;
    dense_plan_kernel<<<static_cast<unsigned>((a.nq + 7) / 8), 256, 0, st>>>(a);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_dense_emit(a, st);
}

// ------------------------------------------------------------ shard protocol
// The sharded select: every shard scores its own points with the two-pass dense
// select's K1, then two exchanges fix the reference's global top-m by (score desc, id asc)
// (query.cpp:242-260): (1) per-shard totals #(score >= t) -> every shard derives the same T and
// need = m - #(score > T); (2) per-block tie counts at T, block-cyclic -> the first `need` ties
// in GLOBAL id order give each block's quota. K3 then emits the shard's candidates.

// exchange 1: tot[q][t - 1] = #local points with score >= t, t = 1..16 (levels past 8 * nc are 0)
__global__ void __launch_bounds__(256) shard_totals_kernel(DenseArgs a, uint32_t* tot) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t q = uint64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (q >= a.nq) return;
    const uint32_t nc = nc_of(a), LV = 8 * nc;
    const uint4* h = reinterpret_cast<const uint4*>(a.hist) + q * a.P * nc;
    uint32_t acc[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) acc[t] = 0;
    for (uint32_t p = lane; p < a.P; p += 32) {
#pragma unroll
        for (uint32_t t = 1; t <= 16; ++t) {
            if (t <= LV) acc[t - 1] += level_n(h + p * nc, t);
        }
    }
#pragma unroll
    for (int t = 0; t < 16; ++t) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[t] += __shfl_xor_sync(kFull, acc[t], o);
    }
    if (lane < 16) {
        uint32_t v = 0;
#pragma unroll
        for (int t = 0; t < 16; ++t) v = lane == static_cast<uint32_t>(t) ? acc[t] : v;
        tot[q * 16 + lane] = v;
    }
}

// T / need from every shard's totals (G x nq x 16), then per LOCAL block the ties at T
// (ties[q][lb], nbl_max columns, zero past this shard's blocks).
__global__ void __launch_bounds__(256) shard_ties_kernel(DenseArgs a, const uint32_t* tot_all, uint32_t G,
                                                         uint64_t n_global, uint32_t ppb, uint32_t nbl,
                                                         uint32_t nbl_max, uint32_t* T_out, uint64_t* need_out,
                                                         uint32_t* ties) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t q = uint64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (q >= a.nq) return;
    const uint32_t nc = nc_of(a), LV = 8 * nc;
    // lane t - 1 holds the global #(score >= t)
    uint64_t ge = 0;
    if (lane < 16) {
        for (uint32_t g = 0; g < G; ++g) ge += tot_all[(uint64_t(g) * a.nq + q) * 16 + lane];
    }
    uint32_t T = 0;
    for (int t = 16; t >= 1; --t) {
        const uint64_t v = __shfl_sync(kFull, ge, t - 1);
        if (T == 0 && static_cast<uint32_t>(t) <= min(a.ns, LV) && v >= a.m) T = t;
    }
    // #(score > T) = #(score >= T + 1); level N_s + 1 and above is empty
    const uint64_t gtT = (T + 1 <= 16) ? __shfl_sync(kFull, ge, T < 16 ? T : 0) : 0;
    const uint64_t gt_total = (T + 1 <= min(a.ns, LV)) ? gtT : 0;
    (void)n_global;
    const uint4* h = reinterpret_cast<const uint4*>(a.hist) + q * a.P * nc;
    for (uint32_t lb = lane; lb < nbl_max; lb += 32) {
        uint32_t t = 0;
        if (lb < nbl) {
            for (uint32_t p = lb * ppb; p < min(a.P, (lb + 1) * ppb); ++p) {
                const uint32_t len = static_cast<uint32_t>(min_u64(a.WP, a.n - uint64_t(p) * a.WP));
                const uint32_t geT = T ? level_n(h + p * nc, T) : len;
                const uint32_t gt = T + 1 <= LV ? level_n(h + p * nc, T + 1) : 0u;
                t += geT - gt;
            }
        }
        ties[q * nbl_max + lb] = t;
    }
    if (lane == 0) {
        T_out[q] = T;
        need_out[q] = a.m - gt_total;
    }
}

// Quotas in global id order (block j of shard j % G, local block j / G), then per local piece:
// quota (first ties of the block's quota, piece order), output offset, and the local count.
__global__ void __launch_bounds__(256) shard_quota_kernel(DenseArgs a, const uint32_t* ties_all, uint32_t G,
                                                          uint32_t shard, uint64_t nb_global, uint32_t ppb,
                                                          uint32_t nbl, uint32_t nbl_max, const uint64_t* need_in,
                                                          uint32_t* qblk, uint32_t* counts) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t q = uint64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (q >= a.nq) return;
    const uint32_t nc = nc_of(a), LV = 8 * nc;
    const uint64_t need = need_in[q];
    uint64_t run = 0;
    for (uint64_t j0 = 0; j0 < nb_global; j0 += 32) {
        const uint64_t j = j0 + lane;
        uint32_t t = 0;
        if (j < nb_global) t = ties_all[(uint64_t(j % G) * a.nq + q) * nbl_max + j / G];
        uint32_t x = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, x, o);
            if (lane >= static_cast<uint32_t>(o)) x += y;
        }
        const uint64_t before = run + x - t;
        const uint32_t quota = before >= need ? 0u : static_cast<uint32_t>(min_u64(t, need - before));
        if (j < nb_global && j % G == shard) qblk[q * nbl_max + j / G] = quota;
        run += __shfl_sync(kFull, x, 31);
    }
    __syncwarp();
    const uint32_t T = a.T[q];
    const uint4* h = reinterpret_cast<const uint4*>(a.hist) + q * a.P * nc;
    uint64_t out_run = 0;
    for (uint32_t lb0 = 0; lb0 < nbl; lb0 += 32) {
        const uint32_t lb = lb0 + lane;
        uint32_t btake = 0;
        if (lb < nbl) {
            uint32_t left = qblk[q * nbl_max + lb];
            for (uint32_t p = lb * ppb; p < min(a.P, (lb + 1) * ppb); ++p) {
                const uint32_t len = static_cast<uint32_t>(min_u64(a.WP, a.n - uint64_t(p) * a.WP));
                const uint32_t geT = T ? level_n(h + p * nc, T) : len;
                const uint32_t gt = T + 1 <= LV ? level_n(h + p * nc, T + 1) : 0u;
                const uint32_t pq = min(geT - gt, left);
                left -= pq;
                a.quota[q * a.P + p] = pq;
                btake += gt + pq;
            }
        }
        uint32_t x = btake;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, x, o);
            if (lane >= static_cast<uint32_t>(o)) x += y;
        }
        if (lb < nbl) {
            uint32_t pos = static_cast<uint32_t>(out_run + x - btake);
            for (uint32_t p = lb * ppb; p < min(a.P, (lb + 1) * ppb); ++p) {
                const uint32_t gt = T + 1 <= LV ? level_n(h + p * nc, T + 1) : 0u;
                a.base[q * a.P + p] = pos;
                pos += gt + a.quota[q * a.P + p];
            }
        }
        out_run += __shfl_sync(kFull, x, 31);
    }
    if (lane == 0) counts[q] = static_cast<uint32_t>(out_run);
}

// ---- the shard protocol's single pass (the unsharded path's K0 / bound / fused pass / plan /
// compaction, with the speculative bound and the tie quotas agreed across shards):
//   S0 every shard's sampled totals (17 u32 per query) -> all-reduce (sum) -> shard_bound_kernel:
//      the same L and the same tie cut (in GLOBAL pieces) on every shard;
//   S1 the fused pass over the shard's pieces (tie cuts compared in global piece order, gpiece);
//   S2 per query #(score > L) of the shard -> all-reduce; per local block the ties counted before
//      the cut -> all-gather;
//   S3 shard_fused_plan_kernel: need = m - #(score > L), the first `need` ties in GLOBAL id order
//      give each block its quota (shard_quota_kernel's rule), split over the block's pieces in id
//      order; offsets (score > L first, then the ties) and the shard's candidate count; a query
//      whose quota reaches past the cut or whose contributing buffer overflowed is flagged, and a
//      flag on any shard sends the whole tile through the two-pass protocol above.
__global__ void __launch_bounds__(256) shard_sample_kernel(DenseArgs a, uint32_t* out) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t q = uint64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (q >= a.nq) return;
    uint32_t tot[16];
    const uint64_t sampled = sample_totals(a, q, lane, tot);
    if (lane < 17) {
        uint32_t v = static_cast<uint32_t>(sampled);
#pragma unroll
        for (int t = 0; t < 16; ++t) v = lane == static_cast<uint32_t>(t) ? tot[t] : v;
        out[q * 17 + lane] = v;
    }
}

__global__ void __launch_bounds__(256) shard_bound_kernel(DenseArgs a, const uint32_t* sum17, uint64_t n_global,
                                                          uint32_t P_global) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t q = uint64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (q >= a.nq) return;
    uint32_t tot[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) tot[t] = sum17[q * 17 + t];
    const Bound b = bound_core(a, tot, sum17[q * 17 + 16], n_global, P_global);
    if (lane == 0) {
        a.L[q] = b.L | (b.dense ? kDenseStage : 0u);
        a.pcut[q] = b.cut;
    }
}

// gt[q] = the shard's #(score > L); ties[q][lb] = its block lb's ties at L counted by the fused pass
// (pieces past every tie cut of their CTA recorded none).
__global__ void __launch_bounds__(256) shard_fused_sums_kernel(DenseArgs a, uint32_t ppb, uint32_t nbl,
                                                               uint32_t nbl_max, uint32_t* gt, uint32_t* ties) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t q = uint64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (q >= a.nq) return;
    const uint32_t* h = a.h2 + q * a.P;
    uint32_t g = 0;
    for (uint32_t lb = lane; lb < nbl_max; lb += 32) {
        uint32_t t = 0;
        if (lb < nbl) {
            for (uint32_t p = lb * ppb; p < min(a.P, (lb + 1) * ppb); ++p) {
                const uint32_t v = h[p];
                g += v >> 16;
                t += (v & 0xffffu) - (v >> 16);
            }
        }
        ties[q * nbl_max + lb] = t;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) g += __shfl_xor_sync(kFull, g, o);
    if (lane == 0) gt[q] = g;
}

__global__ void __launch_bounds__(256) shard_fused_plan_kernel(DenseArgs a, const uint32_t* gt_sum, const uint32_t* gt_local,
                                                               const uint32_t* ties_all, uint32_t G, uint32_t shard,
                                                               uint64_t nb_global, uint32_t ppb, uint32_t nbl,
                                                               uint32_t nbl_max, uint32_t* qblk, uint32_t* counts,
                                                               uint32_t* nflag) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t q = uint64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (q >= a.nq) return;
    const uint32_t L = a.L[q] & 0xffu;
    const uint64_t geL1 = gt_sum[q];  // global #(score > L)
    bool ok = L >= 1 && geL1 < a.m;
    const uint64_t need = ok ? a.m - geL1 : 0;
    // block quotas in global id order (block j on shard j % G, local block j / G)
    uint64_t run = 0;
    for (uint64_t j0 = 0; j0 < nb_global; j0 += 32) {
        const uint64_t j = j0 + lane;
        const uint32_t t = j < nb_global ? ties_all[(uint64_t(j % G) * a.nq + q) * nbl_max + j / G] : 0u;
        uint32_t x = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, x, o);
            if (lane >= static_cast<uint32_t>(o)) x += y;
        }
        const uint64_t before = run + x - t;
        const uint32_t quota = before >= need ? 0u : static_cast<uint32_t>(min_u64(t, need - before));
        if (j < nb_global && j % G == shard) qblk[q * nbl_max + j / G] = quota;
        run += __shfl_sync(kFull, x, 31);
    }
    ok = ok && run >= need;  // the ties counted before the cuts cover the quota
    __syncwarp();
    // per local block (lane), its pieces in id order: quotas, the two offsets, the checks
    const uint32_t* h = a.h2 + q * a.P;
    const uint64_t gl = gt_local[q];
    uint64_t gt_run = 0, tie_run = 0;
    for (uint32_t lb0 = 0; lb0 < nbl; lb0 += 32) {
        const uint32_t lb = lb0 + lane;
        uint32_t bgt = 0, btie = 0;
        if (lb < nbl) {
            uint32_t left = qblk[q * nbl_max + lb];
            for (uint32_t p = lb * ppb; p < min(a.P, (lb + 1) * ppb); ++p) {
                const uint32_t v = h[p];
                const uint32_t gt = v >> 16, ties = (v & 0xffffu) - gt;
                const uint32_t pq = min(ties, left);
                left -= pq;
                a.quota[q * a.P + p] = pq;
                if (pq && gpiece(a, p) >= a.pcut[q]) ok = false;           // ties needed past the tie cut
                if ((gt + pq) && a.ccnt[q * a.P + p] > a.B) ok = false;   // a contributing buffer overflowed
                bgt += gt;
                btie += pq;
            }
        }
        uint32_t xg = bgt, xt = btie;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, xg, o), z = __shfl_up_sync(kFull, xt, o);
            if (lane >= static_cast<uint32_t>(o)) {
                xg += y;
                xt += z;
            }
        }
        if (lb < nbl) {
            uint32_t pg = static_cast<uint32_t>(gt_run + xg - bgt), pt = static_cast<uint32_t>(gl + tie_run + xt - btie);
            for (uint32_t p = lb * ppb; p < min(a.P, (lb + 1) * ppb); ++p) {
                a.base[q * a.P + p] = pg;
                a.base2[q * a.P + p] = pt;
                pg += h[p] >> 16;
                pt += a.quota[q * a.P + p];
            }
        }
        gt_run += __shfl_sync(kFull, xg, 31);
        tie_run += __shfl_sync(kFull, xt, 31);
    }
    ok = __all_sync(kFull, ok);
    if (lane == 0) {
        a.qflag[q] = ok ? 0u : 1u;
        a.T[q] = L;
        counts[q] = static_cast<uint32_t>(gl + tie_run);
        if (!ok) atomicAdd(nflag, 1u);
        if (ok && a.clist) {  // the compaction kernels' work lists
            const uint32_t wl = dense_compact_warp(a, q) ? 0u : 1u;
            a.clist[wl * a.nq + atomicAdd(a.nclist + wl, 1u)] = static_cast<uint32_t>(q);
        }
    }
}

cudaError_t launch_shard_sample(const DenseArgs& a, uint32_t* sum17, cudaStream_t st) {
    if (a.nq == 0) return cudaSuccess;
    cudaError_t e = launch_dense_sample(a, st);
    if (e != cudaSuccess) return e;
    shard_sample_kernel<<<static_cast<unsigned>((a.nq + 7) / 8), 256, 0, st>>>(a, sum17);
    return cudaGetLastError();
}

cudaError_t launch_shard_bound(const DenseArgs& a, const uint32_t* sum17, uint64_t n_global, uint32_t P_global,
                               cudaStream_t st) {
    if (a.nq == 0) return cudaSuccess;
    shard_bound_kernel<<<static_cast<unsigned>((a.nq + 7) / 8), 256, 0, st>>>(a, sum17, n_global, P_global);
    return cudaGetLastError();
}

cudaError_t launch_shard_fused_sums(const DenseArgs& a, uint32_t ppb, uint32_t nbl, uint32_t nbl_max, uint32_t* gt,
                                    uint32_t* ties, cudaStream_t st) {
    if (a.nq == 0) return cudaSuccess;
    shard_fused_sums_kernel<<<static_cast<unsigned>((a.nq + 7) / 8), 256, 0, st>>>(a, ppb, nbl, nbl_max, gt, ties);
    return cudaGetLastError();
}

cudaError_t launch_shard_fused_plan(const DenseArgs& a, const uint32_t* gt_sum, const uint32_t* gt_local,
                                    const uint32_t* ties_all, uint32_t G, uint32_t shard, uint64_t nb_global,
                                    uint32_t ppb, uint32_t nbl, uint32_t nbl_max, uint32_t* qblk, uint32_t* counts,
                                    uint32_t* nflag, cudaStream_t st) {
    if (a.nq == 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(a.nclist, 0, 2 * sizeof(uint32_t), st);
    if (e != cudaSuccess) return e;
    shard_fused_plan_kernel<<<static_cast<unsigned>((a.nq + 7) / 8), 256, 0, st>>>(
        a, gt_sum, gt_local, ties_all, G, shard, nb_global, ppb, nbl, nbl_max, qblk, counts, nflag);
    return cudaGetLastError();
}

cudaError_t launch_shard_totals(const DenseArgs& a, uint32_t* tot, cudaStream_t st) {
    if (a.nq == 0) return cudaSuccess;
    shard_totals_kernel<<<static_cast<unsigned>((a.nq + 7) / 8), 256, 0, st>>>(a, tot);
    return cudaGetLastError();
}

cudaError_t launch_shard_ties(const DenseArgs& a, const uint32_t* tot_all, uint32_t G, uint32_t ppb, uint32_t nbl,
                              uint32_t nbl_max, uint32_t* T, uint64_t* need, uint32_t* ties, cudaStream_t st) {
    if (a.nq == 0) return cudaSuccess;
    shard_ties_kernel<<<static_cast<unsigned>((a.nq + 7) / 8), 256, 0, st>>>(a, tot_all, G, 0, ppb, nbl, nbl_max, T,
                                                                              need, ties);
    return cudaGetLastError();
}

cudaError_t launch_shard_quota(const DenseArgs& a, const uint32_t* ties_all, uint32_t G, uint32_t shard,
                               uint64_t nb_global, uint32_t ppb, uint32_t nbl, uint32_t nbl_max, const uint64_t* need,
                               uint32_t* qblk, uint32_t* counts, cudaStream_t st) {
    if (a.nq == 0) return cudaSuccess;
    shard_quota_kernel<<<static_cast<unsigned>((a.nq + 7) / 8), 256, 0, st>>>(a, ties_all, G, shard, nb_global, ppb,
                                                                               nbl, nbl_max, need, qblk, counts);
    return cudaGetLastError();
}

}  // namespace suco_gpu
