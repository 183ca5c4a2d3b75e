// SC-Linear on the GPU: the index-free baseline / quality
// oracle of sc_linear.cpp:49-121, bit-identical to it, over a BATCH of queries.
//
//   compute_sc_scores (sc_linear.cpp:49-93): per subspace, the exact fp64
//   squared distance of every point's whole-subspace projection to the
//   query's, then the collision_count(alpha, n) smallest by (distance, id)
//   each score one collision;
//   sc_linear_query (:95-121): the candidate_count(beta, n, k) best by
//   (score desc, id asc), re-ranked exactly (the query path's kernels).
//
// The distance follows the reference's two code paths exactly: a subspace
// whose dims are one consecutive run goes through sq_euclidean_raw (four
// strided accumulators, core.hpp:66-84); any other through
// sq_euclidean_projected (one sequential accumulator, subspace.cpp:105-121).
//
// Top-c per (query, subspace) is a hand-written MSB radix select on the
// distance bit patterns (non-negative doubles order like their bits): six
// passes of 11-bit digits, each a shared-memory histogram per CTA chunk merged
// with global atomics, find the c-th distance D and how many lie below it;
// the ties at D are taken lowest ids first (the reference's nth_element order
// on (distance, id), a strict total order) from per-chunk tie counts and their
// prefix. Scores are u8 (<= N_s). The m candidates follow the same scheme on
// the scores: a 256-bin histogram, the threshold score, and the id-ordered
// tie prefix.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.h"

namespace suco_gpu {
namespace {

constexpr uint32_t kScChunk = 4096;  // points per CTA chunk (tie counts, emission)
constexpr uint32_t kScBins = 2048;   // 11-bit digits

__global__ void __launch_bounds__(256) sc_dist_kernel(ScArgs a, uint32_t s) {
    const uint32_t b = blockIdx.y;
    const float* q = a.q + uint64_t(b) * a.d;
    unsigned long long* keys = a.keys + uint64_t(b) * a.n;
    const uint32_t off = a.sub_off[s], len = a.sub_off[s + 1] - off;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < a.n; i += uint64_t(gridDim.x) * blockDim.x) {
        const float* row = a.data + i * a.d;
        double dist;
        if (a.consec[s]) {  // sq_euclidean_raw over data[start, start + len)
            const float* x = row + a.dims[off];
            const float* qq = q + a.dims[off];
            double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
            uint32_t j = 0;
            for (; j + 4 <= len; j += 4) {
                const double d0 = __dsub_rn(double(x[j]), double(qq[j]));
                const double d1 = __dsub_rn(double(x[j + 1]), double(qq[j + 1]));
                const double d2 = __dsub_rn(double(x[j + 2]), double(qq[j + 2]));
                const double d3 = __dsub_rn(double(x[j + 3]), double(qq[j + 3]));
                acc0 = __dadd_rn(acc0, __dmul_rn(d0, d0));
                acc1 = __dadd_rn(acc1, __dmul_rn(d1, d1));
                acc2 = __dadd_rn(acc2, __dmul_rn(d2, d2));
                acc3 = __dadd_rn(acc3, __dmul_rn(d3, d3));
            }
            for (; j < len; ++j) {
                const double dd = __dsub_rn(double(x[j]), double(qq[j]));
                acc0 = __dadd_rn(acc0, __dmul_rn(dd, dd));
            }
            dist = __dadd_rn(__dadd_rn(acc0, acc1), __dadd_rn(acc2, acc3));
        } else {  // sq_euclidean_projected: dims in layout order, one accumulator
            double acc = 0.0;
            for (uint32_t j = 0; j < len; ++j) {
                const uint32_t dim = a.dims[off + j];
                const double dd = __dsub_rn(double(row[dim]), double(q[dim]));
                acc = __dadd_rn(acc, __dmul_rn(dd, dd));
            }
            dist = acc;
        }
        keys[i] = static_cast<unsigned long long>(__double_as_longlong(dist));
    }
}

// Radix select state per query: prefix / mask of the bucket holding rank `need`, elements below it.
struct RxState {
    unsigned long long prefix, mask;
    uint64_t need, below;
};

__global__ void sc_rx_init_kernel(RxState* st, uint32_t B, uint64_t c) {
    const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < B) st[b] = RxState{0ull, 0ull, c, 0};
}

// one 11-bit digit (bits [shift, shift + 11) & 63) of every key in the query's current bucket
__global__ void __launch_bounds__(256) sc_rx_hist_kernel(const unsigned long long* keys, uint64_t n,
                                                         const RxState* st, uint32_t shift, uint32_t* hist) {
    __shared__ uint32_t h[kScBins];
    const uint32_t b = blockIdx.y;
    for (uint32_t i = threadIdx.x; i < kScBins; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const RxState s = st[b];
    const unsigned long long* kb = keys + uint64_t(b) * n;
    const uint64_t lo = uint64_t(blockIdx.x) * kScChunk, hi = min_u64(n, lo + kScChunk);
    for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const unsigned long long u = kb[i];
        if ((u & s.mask) == s.prefix) atomicAdd(&h[(u >> shift) & (kScBins - 1)], 1u);
    }
    __syncthreads();
    uint32_t* gh = hist + uint64_t(b) * kScBins;
    for (uint32_t i = threadIdx.x; i < kScBins; i += blockDim.x) {
        if (h[i]) atomicAdd(gh + i, h[i]);
    }
}

// the bin holding rank `need` (one CTA per query), then the histogram is cleared for the next pass
__global__ void __launch_bounds__(256) sc_rx_pick_kernel(RxState* st, uint32_t* hist, uint32_t shift, uint32_t bits) {
    __shared__ uint32_t part[256];
    const uint32_t b = blockIdx.x, t = threadIdx.x;
    uint32_t* h = hist + uint64_t(b) * kScBins;
    uint32_t loc[kScBins / 256], sum = 0;
#pragma unroll
    for (uint32_t j = 0; j < kScBins / 256; ++j) {
        loc[j] = h[t * (kScBins / 256) + j];
        sum += loc[j];
    }
    part[t] = sum;
    __syncthreads();
    if (t == 0) {  // exclusive prefix over the 256 parts
        uint32_t run = 0;
        for (uint32_t i = 0; i < 256; ++i) {
            const uint32_t v = part[i];
            part[i] = run;
            run += v;
        }
    }
    __syncthreads();
    RxState s = st[b];
    const uint64_t need = s.need;
    uint32_t run = part[t];
#pragma unroll
    for (uint32_t j = 0; j < kScBins / 256; ++j) {
        if (run < need && need <= uint64_t(run) + loc[j]) {  // exactly one bin holds rank `need`
            s.prefix |= static_cast<unsigned long long>(t * (kScBins / 256) + j) << shift;
            s.mask |= ((1ull << bits) - 1ull) << shift;
            s.below += run;
            s.need = need - run;
            st[b] = s;
        }
        run += loc[j];
    }
    __syncthreads();
#pragma unroll
    for (uint32_t j = 0; j < kScBins / 256; ++j) h[t * (kScBins / 256) + j] = 0;
}

// per chunk: how many keys equal the c-th key (ties at D)
__global__ void __launch_bounds__(256) sc_tie_count_kernel(const unsigned long long* keys, uint64_t n,
                                                           const RxState* st, uint32_t nchunks, uint32_t* tcount) {
    __shared__ uint32_t cnt;
    const uint32_t b = blockIdx.y;
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    const unsigned long long D = st[b].prefix;
    const unsigned long long* kb = keys + uint64_t(b) * n;
    const uint64_t lo = uint64_t(blockIdx.x) * kScChunk, hi = min_u64(n, lo + kScChunk);
    uint32_t c = 0;
    for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) c += kb[i] == D;
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31u) == 0 && c) atomicAdd(&cnt, c);
    __syncthreads();
    if (threadIdx.x == 0) tcount[uint64_t(b) * nchunks + blockIdx.x] = cnt;
}

// exclusive prefix of the chunk tie counts (one CTA per query, chunks in id order)
__global__ void __launch_bounds__(256) sc_prefix_kernel(uint32_t* v, uint32_t nchunks) {
    __shared__ uint32_t carry;
    const uint32_t b = blockIdx.x, t = threadIdx.x;
    uint32_t* row = v + uint64_t(b) * nchunks;
    if (t == 0) carry = 0;
    __syncthreads();
    for (uint32_t base = 0; base < nchunks; base += 256) {
        const uint32_t i = base + t;
        const uint32_t x = i < nchunks ? row[i] : 0u;
        uint32_t incl = x;
        const uint32_t lane = t & 31u, warp = t >> 5;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= static_cast<uint32_t>(o)) incl += y;
        }
        __shared__ uint32_t wsum[8];
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        uint32_t woff = 0;
        for (uint32_t w = 0; w < warp; ++w) woff += wsum[w];
        const uint32_t c0 = carry;
        if (i < nchunks) row[i] = c0 + woff + incl - x;
        __syncthreads();
        if (t == 255) carry = c0 + woff + incl;
        __syncthreads();
    }
}

// score += 1 for the top c: key < D, or key == D among the first (c - below) ties in id order
__global__ void __launch_bounds__(256) sc_mark_kernel(const unsigned long long* keys, uint64_t n, const RxState* st,
                                                      uint32_t nchunks, const uint32_t* tprefix, uint8_t* scores) {
    __shared__ uint32_t wtie[8];
    const uint32_t b = blockIdx.y;
    const RxState s = st[b];
    const unsigned long long D = s.prefix;
    const uint64_t take = s.need;  // ties to take overall (need after the last pass: rank inside the ties)
    const unsigned long long* kb = keys + uint64_t(b) * n;
    uint8_t* sc = scores + uint64_t(b) * n;
    const uint64_t lo = uint64_t(blockIdx.x) * kScChunk, hi = min_u64(n, lo + kScChunk);
    uint64_t seen = tprefix[uint64_t(b) * nchunks + blockIdx.x];  // ties before this chunk
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    for (uint64_t base = lo; base < hi; base += blockDim.x) {
        const uint64_t i = base + threadIdx.x;
        const unsigned long long u = i < hi ? kb[i] : ~0ull;
        const bool tie = i < hi && u == D;
        const uint32_t bal = __ballot_sync(0xffffffffu, tie);
        if (lane == 0) wtie[warp] = __popc(bal);
        __syncthreads();
        uint32_t before = 0, total = 0;
        for (uint32_t w = 0; w < 8; ++w) {
            before += w < warp ? wtie[w] : 0u;
            total += wtie[w];
        }
        const uint64_t rank = seen + before + __popc(bal & ((1u << lane) - 1u));  // ties before this one
        if (i < hi && (u < D || (tie && rank < take))) sc[i] += 1;
        seen += total;
        __syncthreads();
    }
}

// scores -> per chunk counts of each score value (u8 histogram, 16 levels kept: N_s <= 255 but
// the candidate plan only needs the levels at and above the threshold; all 256 are counted)
__global__ void __launch_bounds__(256) sc_score_hist_kernel(const uint8_t* scores, uint64_t n, uint32_t* hist) {
    __shared__ uint32_t h[256];
    const uint32_t b = blockIdx.y;
    h[threadIdx.x] = 0;
    __syncthreads();
    const uint8_t* sc = scores + uint64_t(b) * n;
    const uint64_t lo = uint64_t(blockIdx.x) * kScChunk, hi = min_u64(n, lo + kScChunk);
    for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) atomicAdd(&h[sc[i]], 1u);
    __syncthreads();
    if (h[threadIdx.x]) atomicAdd(hist + uint64_t(b) * 256 + threadIdx.x, h[threadIdx.x]);
}

// T = max{t : #(score >= t) >= m} and need = m - #(score > T), per query (one warp... one thread)
__global__ void sc_score_plan_kernel(const uint32_t* hist, uint32_t B, uint64_t m, RxState* st) {
    const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    const uint32_t* h = hist + uint64_t(b) * 256;
    uint64_t ge = 0;
    uint32_t T = 0;
    uint64_t gt = 0;
    for (int t = 255; t >= 0; --t) {
        const uint64_t g2 = ge + h[t];
        if (g2 >= m) {
            T = static_cast<uint32_t>(t);
            gt = ge;
            break;
        }
        ge = g2;
    }
    st[b] = RxState{T, 0ull, m - gt, gt};
}

// per chunk: #score == T (ties) and #score > T (taken), for the emission offsets
__global__ void __launch_bounds__(256) sc_cand_count_kernel(const uint8_t* scores, uint64_t n, const RxState* st,
                                                            uint32_t nchunks, uint32_t* tcount, uint32_t* gcount) {
    __shared__ uint32_t ct, cg;
    const uint32_t b = blockIdx.y;
    if (threadIdx.x == 0) ct = cg = 0;
    __syncthreads();
    const uint32_t T = static_cast<uint32_t>(st[b].prefix);
    const uint8_t* sc = scores + uint64_t(b) * n;
    const uint64_t lo = uint64_t(blockIdx.x) * kScChunk, hi = min_u64(n, lo + kScChunk);
    uint32_t t = 0, g = 0;
    for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        t += sc[i] == T;
        g += sc[i] > T;
    }
    for (int o = 16; o > 0; o >>= 1) {
        t += __shfl_xor_sync(0xffffffffu, t, o);
        g += __shfl_xor_sync(0xffffffffu, g, o);
    }
    if ((threadIdx.x & 31u) == 0) {
        if (t) atomicAdd(&ct, t);
        if (g) atomicAdd(&cg, g);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        tcount[uint64_t(b) * nchunks + blockIdx.x] = ct;
        gcount[uint64_t(b) * nchunks + blockIdx.x] = cg;
    }
}

// emission in id order: every score > T, and the first `need` score == T; the candidate SET of
// sc_linear_query (its order is irrelevant to the re-rank), written at chunk offsets
// gprefix + min(tprefix, need)
__global__ void __launch_bounds__(256) sc_emit_kernel(const uint8_t* scores, uint64_t n, const RxState* st,
                                                      uint32_t nchunks, const uint32_t* tprefix,
                                                      const uint32_t* gprefix, uint64_t m, uint32_t* cands) {
    __shared__ uint32_t wt[8], wg[8];
    const uint32_t b = blockIdx.y;
    const uint32_t T = static_cast<uint32_t>(st[b].prefix);
    const uint64_t need = st[b].need;
    const uint8_t* sc = scores + uint64_t(b) * n;
    uint32_t* out = cands + uint64_t(b) * m;
    const uint64_t lo = uint64_t(blockIdx.x) * kScChunk, hi = min_u64(n, lo + kScChunk);
    uint64_t tseen = tprefix[uint64_t(b) * nchunks + blockIdx.x];
    uint64_t pos = gprefix[uint64_t(b) * nchunks + blockIdx.x] + (tseen < need ? tseen : need);
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    for (uint64_t base = lo; base < hi; base += blockDim.x) {
        const uint64_t i = base + threadIdx.x;
        const uint32_t v = i < hi ? sc[i] : 0u;
        const bool tie = i < hi && v == T, gt = i < hi && v > T;
        const uint32_t bt = __ballot_sync(0xffffffffu, tie), bg = __ballot_sync(0xffffffffu, gt);
        if (lane == 0) {
            wt[warp] = __popc(bt);
            wg[warp] = __popc(bg);
        }
        __syncthreads();
        uint32_t tb = 0, gb = 0, ttot = 0, gtot = 0;
        for (uint32_t w = 0; w < 8; ++w) {
            tb += w < warp ? wt[w] : 0u;
            gb += w < warp ? wg[w] : 0u;
            ttot += wt[w];
            gtot += wg[w];
        }
        const uint64_t trank = tseen + tb + __popc(bt & ((1u << lane) - 1u));
        const uint32_t grank = gb + __popc(bg & ((1u << lane) - 1u));
        // output slot: the > T and the taken ties of this chunk interleave in id order
        if (gt || (tie && trank < need)) {
            const uint64_t ties_before = (trank < need ? trank : need) - (tseen < need ? tseen : need);
            const uint64_t gts_before = grank;
            out[pos + ties_before + gts_before] = static_cast<uint32_t>(i);
        }
        const uint64_t taken = (tseen + ttot < need ? tseen + ttot : need) - (tseen < need ? tseen : need);
        pos += taken + gtot;
        tseen += ttot;
        __syncthreads();
    }
}

}  // namespace

static uint64_t al256(uint64_t x) { return (x + 255) / 256 * 256; }

size_t sc_batch_bytes(uint64_t n, uint32_t B, uint64_t m) {
    (void)m;
    const uint64_t nchunks = (n + kScChunk - 1) / kScChunk;
    return al256(uint64_t(B) * n * 8) + al256(uint64_t(B) * kScBins * 4) + al256(uint64_t(B) * 256 * 4) +
           3 * al256(uint64_t(B) * nchunks * 4) + al256(uint64_t(B) * sizeof(RxState)) + al256(uint64_t(B) * n);
}

cudaError_t launch_sc_batch(ScArgs a, uint32_t B, uint64_t c, uint64_t m, uint32_t* cands, uint8_t* scores_out,
                            cudaStream_t st) {
    const uint32_t nchunks = static_cast<uint32_t>((a.n + kScChunk - 1) / kScChunk);
    // scratch carve-up (a.scratch holds sc_batch_bytes(n, B, m))
    unsigned char* p = static_cast<unsigned char*>(a.scratch);
    auto take = [&](uint64_t bytes) {
        unsigned char* r = p;
        p += al256(bytes);
        return r;
    };
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(take(uint64_t(B) * a.n * 8));
    uint32_t* hist = reinterpret_cast<uint32_t*>(take(uint64_t(B) * kScBins * 4));
    uint32_t* shist = reinterpret_cast<uint32_t*>(take(uint64_t(B) * 256 * 4));
    uint32_t* tcount = reinterpret_cast<uint32_t*>(take(uint64_t(B) * nchunks * 4));
    uint32_t* gcount = reinterpret_cast<uint32_t*>(take(uint64_t(B) * nchunks * 4));
    take(uint64_t(B) * nchunks * 4);  // (spare)
    RxState* rs = reinterpret_cast<RxState*>(take(uint64_t(B) * sizeof(RxState)));
    uint8_t* scores = scores_out ? scores_out : reinterpret_cast<uint8_t*>(take(uint64_t(B) * a.n));
    a.keys = keys;
    cudaError_t e = cudaMemsetAsync(scores, 0, uint64_t(B) * a.n, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(hist, 0, uint64_t(B) * kScBins * 4, st);
    if (e != cudaSuccess) return e;
    const dim3 gdist(static_cast<unsigned>(min_u64((a.n + 255) / 256, 148ull * 8)), B);
    const dim3 gchunk(nchunks, B);
    for (uint32_t s = 0; s < a.ns; ++s) {
        sc_dist_kernel<<<gdist, 256, 0, st>>>(a, s);
        sc_rx_init_kernel<<<(B + 255) / 256, 256, 0, st>>>(rs, B, c);
        // digits: bits 53-63, 42-52, 31-41, 20-30, 9-19, then 0-8 (the hist kernel's 11-bit bin of
        // the last pass includes bits 9-10, equal within the bucket by then)
        const uint32_t shifts[6] = {53, 42, 31, 20, 9, 0}, widths[6] = {11, 11, 11, 11, 11, 9};
        for (uint32_t j = 0; j < 6; ++j) {
            sc_rx_hist_kernel<<<gchunk, 256, 0, st>>>(keys, a.n, rs, shifts[j], hist);
            sc_rx_pick_kernel<<<B, 256, 0, st>>>(rs, hist, shifts[j], widths[j]);
        }
        sc_tie_count_kernel<<<gchunk, 256, 0, st>>>(keys, a.n, rs, nchunks, tcount);
        sc_prefix_kernel<<<B, 256, 0, st>>>(tcount, nchunks);
        sc_mark_kernel<<<gchunk, 256, 0, st>>>(keys, a.n, rs, nchunks, tcount, scores);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    if (!cands) return cudaSuccess;
    e = cudaMemsetAsync(shist, 0, uint64_t(B) * 256 * 4, st);
    if (e != cudaSuccess) return e;
    sc_score_hist_kernel<<<gchunk, 256, 0, st>>>(scores, a.n, shist);
    sc_score_plan_kernel<<<(B + 255) / 256, 256, 0, st>>>(shist, B, m, rs);
    sc_cand_count_kernel<<<gchunk, 256, 0, st>>>(scores, a.n, rs, nchunks, tcount, gcount);
    sc_prefix_kernel<<<B, 256, 0, st>>>(tcount, nchunks);
    sc_prefix_kernel<<<B, 256, 0, st>>>(gcount, nchunks);
    sc_emit_kernel<<<gchunk, 256, 0, st>>>(scores, a.n, rs, nchunks, tcount, gcount, m, cands);
    return cudaGetLastError();
}

}  // namespace suco_gpu
