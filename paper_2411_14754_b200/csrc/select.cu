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
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace suco_gpu {
namespace {

constexpr uint32_t kThreads = 512;
constexpr uint32_t kWarps = kThreads / 32;
constexpr uint32_t kCap = 1024;  // retrieved cells staged per chunk
constexpr uint32_t kFull = 0xffffffffu;
constexpr uint32_t kChAlign = 4 * 32 * kWarps;  // CH multiple of this: whole words per lane-step
constexpr uint32_t kChMax = 100 * 2048;         // 200 KiB of counters per CTA at most

__host__ __device__ inline uint32_t hist_stride(uint32_t ns) { return ns + 2; }

// #bytes of w that are >= t (bytes <= 127, 1 <= t <= 128): SWAR high-bit test.
__device__ __forceinline__ uint32_t swar_ge(uint32_t w, uint32_t t) {
    return __popc((w + (0x80u - t) * 0x01010101u) & 0x80808080u);
}

__device__ __forceinline__ uint32_t bytes_ge(uint32_t w, uint32_t t, bool swar) {
    if (t == 0) return 4;
    if (swar) return swar_ge(w, t);
    uint32_t c = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) c += ((w >> (8 * b)) & 0xffu) >= t;
    return c;
}

struct Smem {
    uint8_t* cnt;        // CH
    uint32_t* hist;      // rounds x hist_stride: [0] = slab length, [t] = #score >= t
    uint32_t* seg_beg;   // kCap
    uint32_t* seg_pre;   // kCap + 1
    uint32_t* wtmp;      // 2 * kWarps
    uint32_t* rquota;    // rounds
    uint32_t* roff;      // rounds
    uint32_t* misc;      // 8
};

__host__ __device__ inline size_t smem_bytes(uint32_t CH, uint32_t rounds, uint32_t ns) {
    return CH + 4ull * (rounds * hist_stride(ns) + kCap + kCap + 1 + 2 * kWarps + 2 * rounds + 8) + 16;
}

__device__ inline Smem carve(unsigned char* base, uint32_t CH, uint32_t rounds, uint32_t ns) {
    Smem s;
    s.cnt = base;
    s.hist = reinterpret_cast<uint32_t*>(base + CH);
    s.seg_beg = s.hist + rounds * hist_stride(ns);
    s.seg_pre = s.seg_beg + kCap;
    s.wtmp = s.seg_pre + kCap + 1;
    s.rquota = s.wtmp + 2 * kWarps;
    s.roff = s.rquota + rounds;
    s.misc = s.roff + rounds;
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

// Counts one slab into s.cnt: cnt[id - lo] = #subspaces whose retrieved
// cells contain id (query.cpp:235-239 restricted to the slab).
__device__ void count_slab(const SelectArgs& a, const Smem& s, uint64_t q, uint32_t slab, uint64_t lo, uint32_t len) {
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    uint4* c4 = reinterpret_cast<uint4*>(s.cnt);
    for (uint32_t i = tid; i < a.CH / 16; i += kThreads) c4[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    if (len == 0) return;
    const uint32_t stride = a.nslabs + 1;
    for (uint32_t sub = 0; sub < a.ns; ++sub) {
        const uint64_t t = q * a.ns + sub;
        const uint32_t nc = a.ncells[t];
        const uint32_t* clist = a.cells + t * a.cells_cap;
        const uint32_t* ids = a.ids + static_cast<uint64_t>(sub) * a.n;
        const uint32_t* soff = a.slab_off + static_cast<uint64_t>(sub) * a.K * stride + slab;
        for (uint32_t c0 = 0; c0 < nc; c0 += kCap) {
            const uint32_t cc = min(kCap, nc - c0);
            // stage the (begin, length) of each retrieved cell's slice in this slab
            uint32_t l0 = 0, l1 = 0;
            const uint32_t i0 = 2 * tid, i1 = 2 * tid + 1;
            if (i0 < cc) {
                const uint32_t* p = soff + static_cast<uint64_t>(__ldg(clist + c0 + i0)) * stride;
                const uint32_t b = __ldg(p), e = __ldg(p + 1);
                s.seg_beg[i0] = b;
                l0 = e - b;
            }
            if (i1 < cc) {
                const uint32_t* p = soff + static_cast<uint64_t>(__ldg(clist + c0 + i1)) * stride;
                const uint32_t b = __ldg(p), e = __ldg(p + 1);
                s.seg_beg[i1] = b;
                l1 = e - b;
            }
            uint32_t total;
            const uint32_t ex = block_excl_scan(l0 + l1, s.wtmp, &total);
            if (i0 < cc) s.seg_pre[i0] = ex;
            if (i1 < cc) s.seg_pre[i1] = ex + l0;
            if (tid == 0) s.seg_pre[cc] = total;
            __syncthreads();
            // flatten: warp w takes ids [total*w/16, total*(w+1)/16)
            const uint32_t fa = static_cast<uint32_t>((static_cast<uint64_t>(total) * warp) / kWarps);
            const uint32_t fb = static_cast<uint32_t>((static_cast<uint64_t>(total) * (warp + 1)) / kWarps);
            uint32_t f = fa + lane;
            // first cell with seg_pre[cur] <= f < seg_pre[cur+1]
            uint32_t lo_i = 0, hi_i = cc;
            if (f < fb) {
                while (hi_i - lo_i > 1) {
                    const uint32_t mid = (lo_i + hi_i) >> 1;
                    if (s.seg_pre[mid] <= f) lo_i = mid;
                    else hi_i = mid;
                }
            }
            uint32_t cur = lo_i;
            for (; f < fb; f += 128) {
                uint32_t pidx[4];
                bool ok[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t g = f + 32u * u;
                    ok[u] = g < fb;
                    pidx[u] = 0;
                    if (ok[u]) {
                        while (s.seg_pre[cur + 1] <= g) ++cur;
                        pidx[u] = s.seg_beg[cur] + (g - s.seg_pre[cur]);
                    }
                }
                uint32_t idv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) idv[u] = ok[u] ? __ldg(ids + pidx[u]) : 0u;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (ok[u]) {
                        const uint32_t l = idv[u] - static_cast<uint32_t>(lo);
                        s.cnt[l] = static_cast<uint8_t>(s.cnt[l] + 1);
                    }
                }
            }
            __syncthreads();
        }
    }
}

// hist[t] = #counters >= t over the slab (t = 1..ns); hist[0] = len.
template <int NSB>
__device__ void slab_histogram(const SelectArgs& a, const Smem& s, uint32_t* hist, uint32_t len) {
    const uint32_t tid = threadIdx.x, lane = tid & 31u;
    if (tid < hist_stride(a.ns)) hist[tid] = tid == 0 ? len : 0u;
    __syncthreads();
    const uint32_t* w32 = reinterpret_cast<const uint32_t*>(s.cnt);
    const uint32_t words = (len + 3) / 4;  // bytes beyond len are zero: they add nothing for t >= 1
    if constexpr (NSB > 0) {
        uint32_t h[NSB];
#pragma unroll
        for (int t = 0; t < NSB; ++t) h[t] = 0;
        for (uint32_t i = tid; i < words; i += kThreads) {
            const uint32_t w = w32[i];
            if (w == 0) continue;
#pragma unroll
            for (int t = 0; t < NSB; ++t) h[t] += swar_ge(w, t + 1);
        }
#pragma unroll
        for (int t = 0; t < NSB; ++t) {
            uint32_t v = h[t];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
            if (lane == 0 && v && (uint32_t)t < a.ns) atomicAdd(hist + t + 1, v);
        }
    } else {
        for (uint32_t i = tid; i < words; i += kThreads) {
            const uint32_t w = w32[i];
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const uint32_t v = (w >> (8 * b)) & 0xffu;
                if (v) atomicAdd(hist + v, 1u);  // exact-value histogram, suffix-summed below
            }
        }
        __syncthreads();
        if (tid == 0) {
            for (uint32_t t = a.ns; t >= 2; --t) hist[t - 1] += hist[t];
        }
    }
    __syncthreads();
}

// Emits this slab's share of the candidate set: every counter > T and the
// first `quota` counters == T, in id order, starting at cands[base].
__device__ void emit_slab(const SelectArgs& a, const Smem& s, uint64_t q, uint64_t lo, uint32_t len, uint32_t T,
                          uint32_t quota, uint32_t base, bool swar) {
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t* w32 = reinterpret_cast<const uint32_t*>(s.cnt);
    const uint32_t words = (len + 3) / 4;
    const uint32_t wpw = (words + kWarps - 1) / kWarps;  // words per warp (contiguous range)
    const uint32_t wa = min(words, warp * wpw), wb = min(words, wa + wpw);
    auto word_counts = [&](uint32_t wi, uint32_t w, uint32_t& g, uint32_t& e) {
        if (wi * 4 + 4 <= len) {
            const uint32_t geT = bytes_ge(w, T, swar), geT1 = bytes_ge(w, T + 1, swar);
            g = geT1;
            e = geT - geT1;
        } else {
            g = e = 0;
            for (uint32_t b = 0; wi * 4 + b < len; ++b) {
                const uint32_t v = (w >> (8 * b)) & 0xffu;
                g += v > T;
                e += v == T;
            }
        }
    };
    // pass A: warp totals
    uint32_t g_tot = 0, e_tot = 0;
    for (uint32_t wi = wa + lane; wi < wb; wi += 32) {
        uint32_t g, e;
        word_counts(wi, w32[wi], g, e);
        g_tot += g;
        e_tot += e;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        g_tot += __shfl_xor_sync(kFull, g_tot, off);
        e_tot += __shfl_xor_sync(kFull, e_tot, off);
    }
    uint32_t tmp;
    const uint32_t g_base = block_excl_scan(lane == 0 ? g_tot : 0u, s.wtmp, &tmp);
    const uint32_t e_base = block_excl_scan(lane == 0 ? e_tot : 0u, s.wtmp, &tmp);
    uint32_t gb = __shfl_sync(kFull, g_base, 0), eb = __shfl_sync(kFull, e_base, 0);
    uint32_t* out = a.cands + q * a.m;
    // pass B: lane-ordered placement within each 32-word step
    for (uint32_t w0 = wa; w0 < wb; w0 += 32) {
        const uint32_t wi = w0 + lane;
        uint32_t w = 0, g = 0, e = 0;
        if (wi < wb) {
            w = w32[wi];
            word_counts(wi, w, g, e);
        }
        uint32_t gx = g, ex = e;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t yg = __shfl_up_sync(kFull, gx, off), ye = __shfl_up_sync(kFull, ex, off);
            if (lane >= (uint32_t)off) {
                gx += yg;
                ex += ye;
            }
        }
        const uint32_t gsum = __shfl_sync(kFull, gx, 31), esum = __shfl_sync(kFull, ex, 31);
        gx -= g;
        ex -= e;
        const uint32_t tie_before = eb + ex;
        uint32_t allow = tie_before >= quota ? 0u : min(e, quota - tie_before);
        uint32_t pos = base + gb + gx + min(tie_before, quota);
        if (g + allow > 0) {
            for (uint32_t b = 0; b < 4 && wi * 4 + b < len; ++b) {
                const uint32_t v = (w >> (8 * b)) & 0xffu;
                if (v > T) {
                    out[pos++] = static_cast<uint32_t>(lo) + wi * 4 + b;
                } else if (v == T && allow > 0) {
                    out[pos++] = static_cast<uint32_t>(lo) + wi * 4 + b;
                    --allow;
                }
            }
        }
        gb += gsum;
        eb += esum;
    }
}

template <int NSB>
__global__ void __launch_bounds__(kThreads, 1) select_kernel(SelectArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    cg::cluster_group cluster = cg::this_cluster();
    const uint32_t rank = cluster.block_rank();
    const uint64_t q = blockIdx.x / a.CS;
    const Smem s = carve(smem, a.CH, a.rounds, a.ns);
    const uint32_t hs = hist_stride(a.ns);
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const bool swar = NSB > 0;

    // pass 1: count + histogram every owned slab
    for (uint32_t r = 0; r < a.rounds; ++r) {
        const uint32_t slab = r * a.CS + rank;
        const uint64_t lo = static_cast<uint64_t>(slab) * a.CH;
        const uint32_t len = slab < a.nslabs ? static_cast<uint32_t>(min_u64(a.CH, a.n - lo)) : 0u;
        count_slab(a, s, q, slab, lo, len);
        if (a.scores_dbg) {
            for (uint32_t i = tid; i < len; i += kThreads) a.scores_dbg[q * a.n + lo + i] = s.cnt[i];
        }
        slab_histogram<NSB>(a, s, s.hist + r * hs, len);
    }
    cluster.sync();

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
    cluster.sync();  // peers finished reading our histograms
    const uint32_t T = s.misc[0];

    for (uint32_t r = 0; r < a.rounds; ++r) {
        const uint32_t slab = r * a.CS + rank;
        if (slab >= a.nslabs) break;
        const uint64_t lo = static_cast<uint64_t>(slab) * a.CH;
        const uint32_t len = static_cast<uint32_t>(min_u64(a.CH, a.n - lo));
        if (a.rounds > 1) count_slab(a, s, q, slab, lo, len);
        emit_slab(a, s, q, lo, len, T, s.rquota[r], s.roff[r], swar);
        __syncthreads();
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

template <int NSB>
cudaError_t launch_select_t(const SelectArgs& a, const SelectConfig& cfg, uint64_t nq, cudaStream_t st) {
    cudaError_t e = cudaFuncSetAttribute(select_kernel<NSB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(cfg.smem));
    if (e != cudaSuccess) return e;
    if (cfg.CS > 8) {
        e = cudaFuncSetAttribute(select_kernel<NSB>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(static_cast<unsigned>(nq * cfg.CS));
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
    return cudaLaunchKernelEx(&lc, select_kernel<NSB>, a);
}

}  // namespace

SelectConfig plan_select(uint64_t n, uint32_t ns, int cluster_size) {
    SelectConfig c;
    c.CS = cluster_size > 0 ? static_cast<uint32_t>(cluster_size) : 8u;
    const uint64_t per = (n + c.CS - 1) / c.CS;
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

cudaError_t launch_select(const SelectArgs& a, const SelectConfig& cfg, uint64_t nq, cudaStream_t st) {
    if (nq == 0) return cudaSuccess;
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
