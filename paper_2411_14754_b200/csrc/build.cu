// Index build on the device: all 2*N_s (subspace, half) k-means jobs at once,
// then the IMI of every subspace by a stable counting sort.
//
// Exactness plan (SURVEY §7 hard parts 1-3), per reference step:
//   project          index.cpp:126-129   gather each half's dims into a
//                                        contiguous n x h job array
//   k-means++        kmeans.cpp:58-114   min_dist update: exact fp64 per point
//                                        (parallel). total/prefix walk: a
//                                        strictly serial fp64 fold on one lane
//                                        (other lanes prefetch), or — when the
//                                        job's data is integer-valued and small
//                                        enough that every partial sum is an
//                                        exact integer < 2^53 — a parallel
//                                        scan, which then gives the identical
//                                        doubles. The RNG stream is replayed on
//                                        the host (mt19937_64(derive_seed)); the
//                                        device consumes a uniform only when
//                                        total > 0, exactly like the reference.
//   assign           kmeans.cpp:19-54    exact fp64 distance to every centroid
//                                        (centroids in smem as doubles), strict
//                                        '<' so ties keep the lower id.
//   update           kmeans.cpp:153-168  stable bucket sort by cluster, then one
//                                        lane per (cluster, dim) folds the sum in
//                                        point order; float(sum * (1/count)).
//   repair           kmeans.cpp:172-188  farthest point from the stale centroid,
//                                        strict '>' (lowest id on ties).
//   build_imi        index.cpp:69-96     stable counting sort by c1*k + c2.
#include <cuda_runtime.h>

#include <cstdlib>
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "build.h"
#include "comm.h"
#include "common.cuh"
#include "kernels.h"

namespace suco_gpu {
namespace {

#define BCUDA(x)                                                                                               \
    do {                                                                                                       \
        const cudaError_t e_ = (x);                                                                            \
        if (e_ != cudaSuccess) raise(SUCO_ERR_INTERNAL, std::string("CUDA error '") + cudaGetErrorString(e_) + \
                                                            "' in " #x);                                       \
    } while (0)

constexpr uint32_t kFull = 0xffffffffu;
constexpr float kInfF = __builtin_huge_valf();

template <typename T>
struct Dev {
    T* p = nullptr;
    size_t n = 0;
    Dev() = default;
    explicit Dev(size_t count) { alloc(count); }
    void alloc(size_t count) {
        release();
        BCUDA(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
        n = count;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    ~Dev() { release(); }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
};

struct KJob {
    uint32_t h;
    uint32_t pad;
    uint64_t off;   // float offset of this job's n x h points
    uint64_t coff;  // float offset of this job's k x h centroids
};

// ------------------------------------------------------------------ project
// rows == nullptr: point i is row i; else row rows[i] (the sampled build's training rows)
__global__ void project_kernel(const float* __restrict__ data, uint64_t n, uint32_t d, const uint32_t* __restrict__ dims,
                               const uint32_t* __restrict__ dim_off, const KJob* __restrict__ jobs, float* __restrict__ proj,
                               const uint32_t* __restrict__ rows) {
    const uint32_t j = blockIdx.y;
    const KJob jb = jobs[j];
    const uint32_t* dl = dims + dim_off[j];
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const float* row = data + (rows ? uint64_t(rows[i]) : i) * d;
        float* out = proj + jb.off + i * jb.h;
        for (uint32_t t = 0; t < jb.h; ++t) out[t] = row[dl[t]];
    }
}

// dst[t] = src[idx[t]] for rows of h floats (the sharded build's column reassembly)
__global__ void gather_rows_kernel(const float* __restrict__ src, const uint32_t* __restrict__ idx, uint64_t n,
                                   uint32_t h, float* __restrict__ dst) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n * h; i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t t = i / h;
        dst[i] = src[uint64_t(idx[t]) * h + i % h];
    }
}

// integer certificate input: any non-integer value, and the largest |value|
__global__ void int_check_kernel(const float* __restrict__ proj, const KJob* __restrict__ jobs, uint64_t n,
                                 unsigned int* nonint, unsigned int* maxabs_bits) {
    const uint32_t j = blockIdx.y;
    const KJob jb = jobs[j];
    const uint64_t cnt = n * jb.h;
    bool bad = false;
    float mx = 0.f;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < cnt; i += uint64_t(gridDim.x) * blockDim.x) {
        const float v = proj[jb.off + i];
        bad |= (v != truncf(v));
        mx = fmaxf(mx, fabsf(v));
    }
    bad = __any_sync(kFull, bad);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, o));
    if ((threadIdx.x & 31) == 0) {
        if (bad) atomicOr(nonint + j, 1u);
        atomicMax(maxabs_bits + j, __float_as_uint(mx));  // non-negative floats order like their bits
    }
}

// ---------------------------------------------------------------- k-means++
__global__ void kpp_init_kernel(double* min_dist, uint8_t* chosen, uint64_t n, uint32_t J) {
    const uint64_t total = n * J;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total; i += uint64_t(gridDim.x) * blockDim.x) {
        min_dist[i] = kInf;
        chosen[i] = 0;
    }
}

// place(): centroid c <- point pick[j]  (kmeans.cpp:64-67)
__global__ void copy_centroid_kernel(const float* proj, const KJob* jobs, const uint32_t* pick, uint32_t c, float* cent) {
    const uint32_t j = blockIdx.x;
    const KJob jb = jobs[j];
    for (uint32_t t = threadIdx.x; t < jb.h; t += blockDim.x) {
        cent[jb.coff + uint64_t(c) * jb.h + t] = proj[jb.off + uint64_t(pick[j]) * jb.h + t];
    }
}

// place(): min_dist[i] = min(min_dist[i], D(x_i, x_pick)), chosen[pick] = 1  (kmeans.cpp:68-72)
__global__ void kpp_update_kernel(const float* __restrict__ proj, const KJob* __restrict__ jobs, uint64_t n,
                                  const uint32_t* __restrict__ pick, double* __restrict__ min_dist, uint8_t* chosen) {
    __shared__ float src[64];
    const uint32_t j = blockIdx.y;
    const KJob jb = jobs[j];
    const uint32_t p = pick[j];
    const float* x = proj + jb.off;
    const bool small = jb.h <= 64;
    if (small) {
        for (uint32_t t = threadIdx.x; t < jb.h; t += blockDim.x) src[t] = x[uint64_t(p) * jb.h + t];
        __syncthreads();
    }
    const float* s = small ? src : x + uint64_t(p) * jb.h;
    double* md = min_dist + uint64_t(j) * n;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const double dist = sqdist4(x + i * jb.h, s, jb.h);
        if (dist < md[i]) md[i] = dist;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) chosen[uint64_t(j) * n + p] = 1;
}

// Chooses the next seed of job blockIdx.x (kmeans.cpp:75-111); one CTA per job.
// prefix[i] receives the running fold; pick is the first i with prefix > target.
__global__ void __launch_bounds__(256) kpp_select_kernel(const float* proj, const KJob* jobs, uint64_t n, uint32_t c,
                                                         const double* __restrict__ min_dist, const uint8_t* chosen,
                                                         const uint8_t* exact, const double* uniforms, uint32_t kmax,
                                                         uint32_t* used, uint32_t* pick, double* prefix_all, float* cent,
                                                         int serial) {
    __shared__ double buf[2][256];
    __shared__ double shd[8];
    __shared__ uint32_t shu[8];
    __shared__ double s_total;
    __shared__ uint32_t s_pick;
    const uint32_t j = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const double* md = min_dist + uint64_t(j) * n;
    double* prefix = prefix_all + uint64_t(j) * n;
    if (exact[j]) {
        // parallel exact prefix, tiles of 256 x 8 elements
        double carry = 0.0;
        for (uint64_t base = 0; base < n; base += 2048) {
            double v[8];
            double loc = 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint64_t i = base + tid * 8 + u;
                v[u] = i < n ? md[i] : 0.0;
                loc += v[u];
            }
            // block exclusive scan of loc
            double x = loc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double y = __shfl_up_sync(kFull, x, o);
                if (lane >= (uint32_t)o) x += y;
            }
            if (lane == 31) shd[warp] = x;
            __syncthreads();
            double wpre = 0.0, tot = 0.0;
            for (uint32_t w = 0; w < 8; ++w) {
                if (w < warp) wpre += shd[w];
                tot += shd[w];
            }
            double run = carry + wpre + (x - loc);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint64_t i = base + tid * 8 + u;
                run += v[u];
                if (i < n) prefix[i] = run;
            }
            carry += tot;
            __syncthreads();
        }
        if (tid == 0) s_total = carry;
    } else if (serial == 0) {
        // The strictly serial fold (kmeans.cpp:77, :83-84) computed exactly in parallel. While the
        // running sum s stays in one binade [2^e, 2^(e+1)), every representable value there is a
        // multiple of U = ulp(s), so fl(s + a) = s + U * rint(a / U) — independent of s except on an
        // exact tie (a / U = m + 1/2, rounded to even) — and the fold is an exact integer prefix sum
        // of rint(a_i / U). Each 2048-value tile is scanned that way up to its first element that
        // crosses into the next binade, is a tie, or meets s == 0 / a subnormal s; that element is
        // added serially (one __dadd_rn) and the scan resumes after it. Crossings are O(log n) per
        // pass, ties rare, so the pass runs at block-scan speed with the serial fold's exact values.
        __shared__ long long wsum[8];
        __shared__ uint32_t s_bad;
        __shared__ double s_run;
        if (tid == 0) s_run = 0.0;
        __syncthreads();
        constexpr double kTwo53 = 9007199254740992.0;
        for (uint64_t base = 0; base < n; base += 2048) {
            const uint32_t len = static_cast<uint32_t>(min_u64(2048, n - base));
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t i = tid * 8 + u;
                v[u] = i < len ? md[base + i] : 0.0;
            }
            uint32_t start = 0;
            while (start < len) {
                const double s0 = s_run;  // exact running sum before element `start`
                const bool tiny = !(s0 >= 2.2250738585072014e-308);  // 0 or subnormal
                const double U = tiny ? 0.0 : ldexp(1.0, ilogb(s0) - 52);  // ulp of s0
                const double S0 = tiny ? 0.0 : s0 / U;  // exact: power-of-two scaling
                // per element: integer increment r (clamped) and a "needs the serial add" flag
                long long r[8];
                bool badv[8];
                long long loc = 0;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint32_t i = tid * 8 + u;
                    const bool live = i >= start && i < len;
                    r[u] = 0;
                    badv[u] = false;
                    if (live) {
                        if (tiny) {
                            badv[u] = v[u] != 0.0;  // 0 + 0 stays exact; anything else goes serial
                        } else {
                            const double q = v[u] / U;  // exact
                            const double m = floor(q);
                            const double f = q - m;  // exact
                            badv[u] = f == 0.5 || q >= 4503599627370496.0;  // tie, or surely crossing
                            const double rr = f > 0.5 ? m + 1.0 : m;
                            r[u] = badv[u] ? 0 : static_cast<long long>(rr);
                        }
                    }
                    loc += r[u];
                }
                // block exclusive scan of the per-thread sums
                long long x = loc;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const long long y = __shfl_up_sync(kFull, x, o);
                    if (lane >= static_cast<uint32_t>(o)) x += y;
                }
                if (lane == 31) wsum[warp] = x;
                if (tid == 0) s_bad = 0xffffffffu;
                __syncthreads();
                long long wpre = 0;
                for (uint32_t w = 0; w < warp; ++w) wpre += wsum[w];
                long long run = wpre + (x - loc);  // exclusive prefix of this thread's first element
                // crossing: S0 + run_before + q >= 2^53 (exact comparisons on integers < 2^53)
                uint32_t first_bad = 0xffffffffu;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint32_t i = tid * 8 + u;
                    if (i >= start && i < len && first_bad == 0xffffffffu) {
                        const double before = S0 + static_cast<double>(run);  // exact while < 2^53
                        if (badv[u] || (!tiny && static_cast<double>(r[u]) + before >= kTwo53) ||
                            (!tiny && before >= kTwo53))
                            first_bad = i;
                        run += r[u];
                    }
                }
                if (first_bad != 0xffffffffu) atomicMin(&s_bad, first_bad);
                __syncthreads();
                const uint32_t bad = s_bad;
                // write the exact prefix of the good elements [start, bad)
                run = wpre + (x - loc);
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint32_t i = tid * 8 + u;
                    if (i >= start && i < len) {
                        run += r[u];
                        if (i < bad) prefix[base + i] = tiny ? s0 : __dmul_rn(S0 + static_cast<double>(run), U);
                    }
                }
                __syncthreads();
                if (bad == 0xffffffffu || bad >= len) {  // the whole rest of the tile was good
                    if (tid == 0) s_run = len > start ? prefix[base + len - 1] : s0;
                    __syncthreads();
                    break;
                }
                // the bad element: its predecessor's exact value, then one serial add
                if (tid == (bad >> 3)) {
                    const double prev = bad > start ? prefix[base + bad - 1] : s0;
                    const double nv = __dadd_rn(prev, v[bad & 7u]);
                    prefix[base + bad] = nv;
                    s_run = nv;
                }
                __syncthreads();
                start = bad + 1;
            }
        }
        if (tid == 0) s_total = s_run;
    } else if (warp == 0) {
        // strictly serial left-to-right fold (kmeans.cpp:77, :83-84): lane 0 adds,
        // the other lanes keep the next 256 values in flight
        double run = 0.0;
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint64_t i = lane + 32u * u;
            v[u] = i < n ? md[i] : 0.0;
        }
        int b = 0;
        for (uint64_t base = 0; base < n; base += 256, b ^= 1) {
#pragma unroll
            for (int u = 0; u < 8; ++u) buf[b][lane + 32 * u] = v[u];
            __syncwarp();
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint64_t i = base + 256 + lane + 32u * u;
                v[u] = i < n ? md[i] : 0.0;
            }
            if (lane == 0) {
                const uint32_t cnt = static_cast<uint32_t>(min_u64(256, n - base));
                for (uint32_t t = 0; t < cnt; ++t) {
                    run = __dadd_rn(run, buf[b][t]);
                    prefix[base + t] = run;
                }
            }
            __syncwarp();
        }
        if (lane == 0) s_total = run;
    }
    __syncthreads();
    const double total = s_total;
    uint32_t p = 0xffffffffu;  // "n" sentinel
    if (total > 0.0) {
        if (tid == 0) {
            const double u = uniforms[uint64_t(j) * kmax + used[j]];
            used[j] += 1;
            const double target = __dmul_rn(u, total);
            uint64_t lo = 0, hi = n;  // first index with prefix > target (prefix is non-decreasing)
            while (lo < hi) {
                const uint64_t mid = (lo + hi) >> 1;
                if (prefix[mid] > target) hi = mid;
                else lo = mid + 1;
            }
            s_pick = lo < n ? static_cast<uint32_t>(lo) : 0xffffffffu;
        }
        __syncthreads();
        p = s_pick;
        if (p == 0xffffffffu) {  // round-off overran the walk: last positive-weight point
            uint32_t best = 0;
            bool found = false;
            for (uint64_t i = tid; i < n; i += blockDim.x) {
                if (md[i] > 0.0) {
                    best = static_cast<uint32_t>(i);
                    found = true;
                }
            }
            uint32_t key = found ? best + 1 : 0;
            for (int o = 16; o > 0; o >>= 1) key = max(key, __shfl_xor_sync(kFull, key, o));
            if (lane == 0) shu[warp] = key;
            __syncthreads();
            if (tid == 0) {
                uint32_t k2 = 0;
                for (int w = 0; w < 8; ++w) k2 = max(k2, shu[w]);
                s_pick = k2 ? k2 - 1 : 0xffffffffu;
            }
            __syncthreads();
            p = s_pick;
        }
    }
    if (p == 0xffffffffu) {  // all remaining points coincide with chosen centroids: lowest unchosen id
        const uint8_t* ch = chosen + uint64_t(j) * n;
        uint32_t best = 0xffffffffu;
        for (uint64_t i = tid; i < n; i += blockDim.x) {
            if (!ch[i]) {
                best = static_cast<uint32_t>(i);
                break;
            }
        }
        for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(kFull, best, o));
        if (lane == 0) shu[warp] = best;
        __syncthreads();
        if (tid == 0) {
            uint32_t b2 = 0xffffffffu;
            for (int w = 0; w < 8; ++w) b2 = min(b2, shu[w]);
            s_pick = b2 == 0xffffffffu ? 0u : b2;
        }
        __syncthreads();
        p = s_pick;
    }
    if (tid == 0) pick[j] = p;
    const KJob jb = jobs[j];
    for (uint32_t t = tid; t < jb.h; t += blockDim.x) cent[jb.coff + uint64_t(c) * jb.h + t] = proj[jb.off + uint64_t(p) * jb.h + t];
}

// ------------------------------------------------------- k-means++ fold over chunks
// The same exact serial fold, spread over the device: each job's min_dist is cut into chunks of
// kKppChunk values. While the running sum s stays in one binade [2^e, 2^(e+1)) a chunk adds exactly
// U * R to it (U = ulp(s), R = sum of rint(a_i / U), an integer), whatever s is inside the binade,
// barring a tie (a_i / U = m + 1/2). So every chunk computes R for the binade its approximate
// prefix (the plain sum of the earlier chunks' sums) lies in — away from the binade's edges — and,
// once its predecessor publishes the exact s_in (decoupled look-back, tickets in chunk-major order
// so a predecessor always runs first), checks s_in is in that binade and s_in / U + R < 2^53:
// then s_out = (s_in / U + R) U exactly. Chunks that cross a binade edge, hold a tie, or start
// near an edge (the first chunks, where s grows through many binades) run the tile-by-tile binade
// scan from s_in (kpp_select_kernel's fold). The pick then needs only the chunk holding the target
// and one exact scan of it. Integer-exact jobs fold by plain sums. Measured at cfg4 (16 jobs x 10M
// values): 20.6 ms per seeding round in one CTA per job ->.
constexpr uint32_t kKppChunk = 32768;

__device__ __forceinline__ double ld_volatile_f64(const double* p) { return *reinterpret_cast<const volatile double*>(p); }

// Exact left-to-right fold of md[lo, hi) continued from s (one CTA, 256 threads, all of them call).
// target >= 0: stops at, and returns in *first, the first index whose running value exceeds target
// (~0ull if none). exact: integer-exact job (plain sums).
__device__ double fold_tiles(const double* md, uint64_t lo, uint64_t hi, double s, bool exact, double target,
                             uint64_t* first) {
    __shared__ long long wsum[8];
    __shared__ double wsd[8];
    __shared__ uint32_t s_bad, s_hit;
    __shared__ double s_run;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    constexpr double kTwo53 = 9007199254740992.0;
    if (tid == 0) s_run = s;
    if (first && tid == 0) *first = ~0ull;
    __syncthreads();
    for (uint64_t base = lo; base < hi; base += 2048) {
        const uint32_t len = static_cast<uint32_t>(min_u64(2048, hi - base));
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t i = tid * 8 + u;
            v[u] = i < len ? md[base + i] : 0.0;
        }
        if (exact) {  // every partial sum an exact integer: a plain block scan
            double loc = 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u) loc += v[u];
            double x = loc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double y = __shfl_up_sync(kFull, x, o);
                if (lane >= static_cast<uint32_t>(o)) x += y;
            }
            if (lane == 31) wsd[warp] = x;
            if (tid == 0) s_hit = 0xffffffffu;
            __syncthreads();
            double wpre = 0.0, tot = 0.0;
            for (uint32_t w = 0; w < 8; ++w) {
                if (w < warp) wpre += wsd[w];
                tot += wsd[w];
            }
            const double s0 = s_run;
            double run = s0 + wpre + (x - loc);
            if (target >= 0.0) {
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    run += v[u];
                    const uint32_t i = tid * 8 + u;
                    if (i < len && run > target) {
                        atomicMin(&s_hit, i);
                        break;
                    }
                }
            }
            __syncthreads();
            if (target >= 0.0 && s_hit != 0xffffffffu) {
                if (tid == 0) *first = base + s_hit;
                __syncthreads();
                return s0;  // (the fold stops at the pick; its value is not needed)
            }
            if (tid == 0) s_run = s0 + tot;
            __syncthreads();
            continue;
        }
        uint32_t start = 0;
        while (start < len) {
            const double s0 = s_run;  // exact running sum before element `start`
            const bool tiny = !(s0 >= 2.2250738585072014e-308);  // 0 or subnormal
            const double U = tiny ? 0.0 : ldexp(1.0, ilogb(s0) - 52);  // ulp of s0
            const double S0 = tiny ? 0.0 : s0 / U;  // exact: power-of-two scaling
            long long r[8];
            bool badv[8];
            long long loc = 0;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t i = tid * 8 + u;
                const bool live = i >= start && i < len;
                r[u] = 0;
                badv[u] = false;
                if (live) {
                    if (tiny) {
                        badv[u] = v[u] != 0.0;  // 0 + 0 stays exact; anything else goes serial
                    } else {
                        const double q = v[u] / U;  // exact
                        const double m = floor(q);
                        const double f = q - m;  // exact
                        badv[u] = f == 0.5 || q >= 4503599627370496.0;  // tie, or surely crossing
                        const double rr = f > 0.5 ? m + 1.0 : m;
                        r[u] = badv[u] ? 0 : static_cast<long long>(rr);
                    }
                }
                loc += r[u];
            }
            long long x = loc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const long long y = __shfl_up_sync(kFull, x, o);
                if (lane >= static_cast<uint32_t>(o)) x += y;
            }
            if (lane == 31) wsum[warp] = x;
            if (tid == 0) {
                s_bad = 0xffffffffu;
                s_hit = 0xffffffffu;
            }
            __syncthreads();
            long long wpre = 0, tot = 0;
            for (uint32_t w = 0; w < 8; ++w) {
                if (w < warp) wpre += wsum[w];
                tot += wsum[w];
            }
            long long run = wpre + (x - loc);  // exclusive prefix of this thread's first element
            uint32_t first_bad = 0xffffffffu;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t i = tid * 8 + u;
                if (i >= start && i < len && first_bad == 0xffffffffu) {
                    const double before = S0 + static_cast<double>(run);  // exact while < 2^53
                    if (badv[u] || (!tiny && static_cast<double>(r[u]) + before >= kTwo53) || (!tiny && before >= kTwo53))
                        first_bad = i;
                    run += r[u];
                }
            }
            if (first_bad != 0xffffffffu) atomicMin(&s_bad, first_bad);
            __syncthreads();
            const uint32_t bad = s_bad;
            run = wpre + (x - loc);
            double prev_bad = s0;  // the exact running value just before `bad` (this thread's copy)
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t i = tid * 8 + u;
                if (i >= start && i < len) {
                    if (i == bad) prev_bad = tiny ? s0 : __dmul_rn(S0 + static_cast<double>(run), U);
                    run += r[u];
                    if (i < bad && target >= 0.0) {
                        const double val = tiny ? s0 : __dmul_rn(S0 + static_cast<double>(run), U);
                        if (val > target) atomicMin(&s_hit, i);
                    }
                }
            }
            if (target >= 0.0 && tid == (bad >> 3) && bad < len) {  // the serial add may be the pick
                const double nv = __dadd_rn(prev_bad, v[bad & 7u]);
                if (nv > target) atomicMin(&s_hit, bad);
            }
            __syncthreads();
            if (target >= 0.0 && s_hit != 0xffffffffu) {
                if (tid == 0) *first = base + s_hit;
                __syncthreads();
                return s0;
            }
            if (bad == 0xffffffffu || bad >= len) {  // the whole rest of the tile was good
                if (tid == 0) s_run = tiny ? s0 : __dmul_rn(S0 + static_cast<double>(tot), U);
                __syncthreads();
                break;
            }
            if (tid == (bad >> 3)) s_run = __dadd_rn(prev_bad, v[bad & 7u]);  // one serial add
            __syncthreads();
            start = bad + 1;
        }
    }
    const double out = s_run;
    __syncthreads();
    return out;
}

// Plain (any-order) sum of each chunk: the approximate prefixes that choose the chunks' binades.
__global__ void __launch_bounds__(256) kpp_chunk_sum_kernel(const double* __restrict__ min_dist, uint64_t n,
                                                            uint32_t NC, double* __restrict__ csum) {
    __shared__ double red[8];
    const uint32_t j = blockIdx.y, c = blockIdx.x, tid = threadIdx.x;
    const uint64_t lo = uint64_t(c) * kKppChunk, hi = min_u64(n, lo + kKppChunk);
    const double* md = min_dist + uint64_t(j) * n;
    double a = 0.0;
    for (uint64_t i = lo + tid; i < hi; i += 256) a += md[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(kFull, a, o);
    if ((tid & 31u) == 0) red[tid >> 5] = a;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += red[w];
        csum[uint64_t(j) * NC + c] = t;
    }
}

// The exact fold chunk by chunk (see above): sin / sout = exact running sums at each chunk's ends.
__global__ void __launch_bounds__(256) kpp_chunk_fold_kernel(const double* __restrict__ min_dist, uint64_t n,
                                                             uint32_t NC, uint32_t J, const uint8_t* exact,
                                                             const double* __restrict__ csum, double* sin, double* sout,
                                                             uint32_t* ready, uint32_t* ticket, uint32_t epoch) {
    __shared__ uint32_t s_t;
    __shared__ double red[8];
    __shared__ long long redi[8];
    __shared__ int redb[8];
    __shared__ double s_in_sh;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    if (tid == 0) s_t = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint32_t c = s_t / J, j = s_t % J;  // chunk-major tickets: a predecessor always holds a smaller one
    const uint64_t lo = uint64_t(c) * kKppChunk, hi = min_u64(n, lo + kKppChunk);
    const double* md = min_dist + uint64_t(j) * n;
    const double* cs = csum + uint64_t(j) * NC;
    const bool ex = exact[j] != 0;
    // approximate prefix of the chunk's start
    double pa = 0.0;
    for (uint32_t c2 = tid; c2 < c; c2 += 256) pa += cs[c2];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pa += __shfl_xor_sync(kFull, pa, o);
    if (lane == 0) red[warp] = pa;
    __syncthreads();
    double P = 0.0;
    for (int w = 0; w < 8; ++w) P += red[w];
    bool slow = true;
    int e = 0;
    long long R = 0;
    if (!ex && c > 0 && P >= 2.2250738585072014e-308) {
        e = ilogb(P);
        const double lo_b = ldexp(1.0, e), hi_b = ldexp(1.0, e + 1);
        const double A = cs[c];
        // away from the binade's edges by far more than the approximate prefix can be off
        slow = !(P >= lo_b * (1.0 + 0x1p-24) && P + A <= hi_b * (1.0 - 0x1p-24));
        if (!slow) {
            const double U = ldexp(1.0, e - 52);
            long long loc = 0;
            bool bad = false;
            for (uint64_t i = lo + tid; i < hi; i += 256) {
                const double q = md[i] / U;
                const double m = floor(q);
                const double f = q - m;
                bad |= f == 0.5 || q >= 4503599627370496.0;
                loc += static_cast<long long>(f > 0.5 ? m + 1.0 : m);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) loc += __shfl_xor_sync(kFull, loc, o);
            const int anyb = __any_sync(kFull, bad);
            if (lane == 0) {
                redi[warp] = loc;
                redb[warp] = anyb;
            }
            __syncthreads();
            for (int w = 0; w < 8; ++w) {
                R += redi[w];
                slow |= redb[w] != 0;
            }
        }
    }
    // look-back: the exact running sum at the chunk's start
    if (tid == 0) {
        double si = 0.0;
        if (c > 0) {
            const volatile uint32_t* rd = ready + uint64_t(j) * NC + c - 1;
            while (*rd != epoch) __nanosleep(32);
            __threadfence();
            si = ld_volatile_f64(sout + uint64_t(j) * NC + c - 1);
        }
        s_in_sh = si;
    }
    __syncthreads();
    const double s_in = s_in_sh;
    double s_out;
    if (ex) {
        s_out = s_in + cs[c];  // integer-exact: every partial sum is exact, any order
    } else if (!slow && s_in >= ldexp(1.0, e) && s_in < ldexp(1.0, e + 1) &&
               s_in / ldexp(1.0, e - 52) + static_cast<double>(R) < 9007199254740992.0) {
        const double U = ldexp(1.0, e - 52);
        s_out = __dmul_rn(s_in / U + static_cast<double>(R), U);  // exact: an integer below 2^53 times U
    } else {
        s_out = fold_tiles(md, lo, hi, s_in, false, -1.0, nullptr);
    }
    if (tid == 0) {
        sin[uint64_t(j) * NC + c] = s_in;
        sout[uint64_t(j) * NC + c] = s_out;
        __threadfence();
        *reinterpret_cast<volatile uint32_t*>(ready + uint64_t(j) * NC + c) = epoch;
    }
}

// The pick of each job (kmeans.cpp:75-111): the first index whose running sum exceeds u * total,
// found in the one chunk that holds it; then the reference's fallbacks (kpp_select_kernel's tail).
__global__ void __launch_bounds__(256) kpp_pick_kernel(const float* proj, const KJob* jobs, uint64_t n, uint32_t c,
                                                       const double* __restrict__ min_dist, const uint8_t* chosen,
                                                       const uint8_t* exact, const double* uniforms, uint32_t kmax,
                                                       uint32_t* used, uint32_t* pick, const double* sin,
                                                       const double* sout, uint32_t NC, float* cent) {
    __shared__ uint32_t shu[8];
    __shared__ uint32_t s_pick, s_chunk;
    __shared__ double s_target;
    __shared__ uint64_t s_first;
    const uint32_t j = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const double* md = min_dist + uint64_t(j) * n;
    const double total = sout[uint64_t(j) * NC + NC - 1];
    uint32_t p = 0xffffffffu;  // "n" sentinel
    if (total > 0.0) {
        if (tid == 0) {
            const double u = uniforms[uint64_t(j) * kmax + used[j]];
            used[j] += 1;
            const double target = __dmul_rn(u, total);
            uint32_t l = 0, h = NC;  // first chunk whose end value exceeds the target
            while (l < h) {
                const uint32_t mid = (l + h) >> 1;
                if (sout[uint64_t(j) * NC + mid] > target) h = mid;
                else l = mid + 1;
            }
            s_chunk = l;
            s_target = target;
        }
        __syncthreads();
        const uint32_t cc = s_chunk;
        if (cc < NC) {
            const uint64_t lo = uint64_t(cc) * kKppChunk, hi = min_u64(n, lo + kKppChunk);
            fold_tiles(md, lo, hi, sin[uint64_t(j) * NC + cc], exact[j] != 0, s_target, &s_first);
            __syncthreads();
            p = s_first != ~0ull ? static_cast<uint32_t>(s_first) : 0xffffffffu;
        }
        if (p == 0xffffffffu) {  // round-off overran the walk: last positive-weight point
            uint32_t best = 0;
            bool found = false;
            for (uint64_t i = tid; i < n; i += blockDim.x) {
                if (md[i] > 0.0) {
                    best = static_cast<uint32_t>(i);
                    found = true;
                }
            }
            uint32_t key = found ? best + 1 : 0;
            for (int o = 16; o > 0; o >>= 1) key = max(key, __shfl_xor_sync(kFull, key, o));
            if (lane == 0) shu[warp] = key;
            __syncthreads();
            if (tid == 0) {
                uint32_t k2 = 0;
                for (int w = 0; w < 8; ++w) k2 = max(k2, shu[w]);
                s_pick = k2 ? k2 - 1 : 0xffffffffu;
            }
            __syncthreads();
            p = s_pick;
        }
    }
    if (p == 0xffffffffu) {  // all remaining points coincide with chosen centroids: lowest unchosen id
        const uint8_t* ch = chosen + uint64_t(j) * n;
        uint32_t best = 0xffffffffu;
        for (uint64_t i = tid; i < n; i += blockDim.x) {
            if (!ch[i]) {
                best = static_cast<uint32_t>(i);
                break;
            }
        }
        for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(kFull, best, o));
        if (lane == 0) shu[warp] = best;
        __syncthreads();
        if (tid == 0) {
            uint32_t b2 = 0xffffffffu;
            for (int w = 0; w < 8; ++w) b2 = min(b2, shu[w]);
            s_pick = b2 == 0xffffffffu ? 0u : b2;
        }
        __syncthreads();
        p = s_pick;
    }
    if (tid == 0) pick[j] = p;
    const KJob jb = jobs[j];
    for (uint32_t t = tid; t < jb.h; t += blockDim.x) cent[jb.coff + uint64_t(c) * jb.h + t] = proj[jb.off + uint64_t(p) * jb.h + t];
}

// ------------------------------------------------------------------- assign
// nearest_centroid (kmeans.cpp:19-33) for every point of every job.
template <int HB>
__global__ void __launch_bounds__(256) assign_kernel(const float* __restrict__ proj, const KJob* __restrict__ jobs,
                                                     uint64_t n, uint32_t k, const float* __restrict__ cent,
                                                     uint32_t* __restrict__ assign) {
    extern __shared__ __align__(16) double cs[];  // k x h centroids as doubles (then as floats: the screen)
    const uint32_t j = blockIdx.y;
    const KJob jb = jobs[j];
    const uint32_t h = jb.h;
    float* cf = reinterpret_cast<float*>(cs + size_t(k) * h);
    for (uint32_t t = threadIdx.x; t < k * h; t += blockDim.x) {
        cs[t] = static_cast<double>(cent[jb.coff + t]);
        if constexpr (HB > 0) cf[t] = cent[jb.coff + t];
    }
    __syncthreads();
    const float* x = proj + jb.off;
    uint32_t* as = assign + uint64_t(j) * n;
    // fp32 screen (HB > 0): FFMA distances f_c; f is within G f + E of the reference's fp64 value
    // (one rounding of x - c, h accumulation roundings), so when the runner-up's lower bound is above
    // the best's upper bound the fp64 argmin is that best — strictly, so the lowest-id tie rule
    // cannot apply. Otherwise (near-ties, overflow) the point takes the exact fp64 loop below.
    const float G = static_cast<float>(2 * h + 8) * 5.9604645e-08f, E = 7.5231638e-37f;  // (2h+8) 2^-24, 2^-120
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        double p[HB > 0 ? HB : 1];
        if constexpr (HB > 0) {
            float pf[HB];
#pragma unroll
            for (int t = 0; t < HB; ++t) pf[t] = t < (int)h ? x[i * h + t] : 0.f;
            float f1 = kInfF, f2 = kInfF;
            uint32_t b1 = 0;
            for (uint32_t c = 0; c < k; ++c) {
                const float* cc = cf + c * h;
                float acc = 0.f;
#pragma unroll
                for (int t = 0; t < HB; ++t) {
                    if ((uint32_t)t < h) {
                        const float e = pf[t] - cc[t];
                        acc = __fmaf_rn(e, e, acc);
                    }
                }
                if (acc < f1) {
                    f2 = f1;
                    f1 = acc;
                    b1 = c;
                } else if (acc < f2) {
                    f2 = acc;
                }
            }
            if (f1 <= 3.0e38f && f2 * (1.f - G) - E > f1 * (1.f + G) + E) {
                as[i] = b1;
                continue;
            }
#pragma unroll
            for (int t = 0; t < HB; ++t) p[t] = static_cast<double>(pf[t]);
        }
        uint32_t best = 0;
        double bd = kInf;
        for (uint32_t c = 0; c < k; ++c) {
            const double* cc = cs + c * h;
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
            uint32_t t = 0;
            if constexpr (HB > 0) {
#pragma unroll
                for (int tt = 0; tt + 4 <= HB; tt += 4) {
                    if ((uint32_t)tt + 4 <= h) {
                        double e0 = __dsub_rn(p[tt], cc[tt]), e1 = __dsub_rn(p[tt + 1], cc[tt + 1]);
                        double e2 = __dsub_rn(p[tt + 2], cc[tt + 2]), e3 = __dsub_rn(p[tt + 3], cc[tt + 3]);
                        a0 = __dadd_rn(a0, __dmul_rn(e0, e0));
                        a1 = __dadd_rn(a1, __dmul_rn(e1, e1));
                        a2 = __dadd_rn(a2, __dmul_rn(e2, e2));
                        a3 = __dadd_rn(a3, __dmul_rn(e3, e3));
                        t = tt + 4;
                    }
                }
#pragma unroll
                for (int tt = 0; tt < HB; ++tt) {
                    if ((uint32_t)tt >= t && (uint32_t)tt < h) {
                        const double e = __dsub_rn(p[tt], cc[tt]);
                        a0 = __dadd_rn(a0, __dmul_rn(e, e));
                    }
                }
            } else {
                const float* xi = x + i * h;
                for (; t + 4 <= h; t += 4) {
                    double e0 = __dsub_rn((double)xi[t], cc[t]), e1 = __dsub_rn((double)xi[t + 1], cc[t + 1]);
                    double e2 = __dsub_rn((double)xi[t + 2], cc[t + 2]), e3 = __dsub_rn((double)xi[t + 3], cc[t + 3]);
                    a0 = __dadd_rn(a0, __dmul_rn(e0, e0));
                    a1 = __dadd_rn(a1, __dmul_rn(e1, e1));
                    a2 = __dadd_rn(a2, __dmul_rn(e2, e2));
                    a3 = __dadd_rn(a3, __dmul_rn(e3, e3));
                }
                for (; t < h; ++t) {
                    const double e = __dsub_rn((double)xi[t], cc[t]);
                    a0 = __dadd_rn(a0, __dmul_rn(e, e));
                }
            }
            const double dist = __dadd_rn(__dadd_rn(a0, a1), __dadd_rn(a2, a3));
            if (dist < bd) {
                bd = dist;
                best = c;
            }
        }
        as[i] = best;
    }
}

// ------------------------------------------------------- stable bucket sort
// J independent problems of n keys < B; chunk = `chunk` consecutive items.
__global__ void bsort_hist_kernel(const uint32_t* __restrict__ keys, uint64_t n, uint32_t B, uint32_t chunk,
                                  uint32_t nch, uint32_t* __restrict__ counts, bool use_smem) {
    extern __shared__ uint32_t hs[];
    const uint32_t j = blockIdx.y, ch = blockIdx.x;
    uint32_t* row = counts + (uint64_t(j) * nch + ch) * B;
    if (use_smem) {
        for (uint32_t b = threadIdx.x; b < B; b += blockDim.x) hs[b] = 0;
        __syncthreads();
    }
    const uint64_t lo = uint64_t(ch) * chunk, hi = min_u64(n, lo + chunk);
    const uint32_t* kk = keys + uint64_t(j) * n;
    for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) atomicAdd(use_smem ? hs + kk[i] : row + kk[i], 1u);
    if (use_smem) {
        __syncthreads();
        for (uint32_t b = threadIdx.x; b < B; b += blockDim.x) row[b] = hs[b];
    }
}

// per (job, bucket): exclusive prefix over chunks; totals per bucket
__global__ void bsort_colscan_kernel(uint32_t* counts, uint32_t B, uint32_t nch, uint32_t J, uint32_t* totals) {
    const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (t >= uint64_t(J) * B) return;
    const uint32_t j = static_cast<uint32_t>(t / B), b = static_cast<uint32_t>(t % B);
    uint32_t run = 0;
    for (uint32_t ch = 0; ch < nch; ++ch) {
        uint32_t* p = counts + (uint64_t(j) * nch + ch) * B + b;
        const uint32_t v = *p;
        *p = run;
        run += v;
    }
    totals[t] = run;
}

// per job: offsets[b] = sum of totals below b; offsets[B] = n
__global__ void bsort_offsets_kernel(const uint32_t* totals, uint32_t B, uint32_t* offsets) {
    __shared__ uint32_t sh[32];
    const uint32_t j = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t* tt = totals + uint64_t(j) * B;
    uint32_t* off = offsets + uint64_t(j) * (B + 1);
    uint32_t carry = 0;
    for (uint32_t b0 = 0; b0 < B; b0 += blockDim.x) {
        const uint32_t b = b0 + tid;
        const uint32_t v = b < B ? tt[b] : 0;
        uint32_t x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, x, o);
            if (lane >= (uint32_t)o) x += y;
        }
        if (lane == 31) sh[warp] = x;
        __syncthreads();
        uint32_t wpre = 0, tot = 0;
        for (uint32_t w = 0; w < (blockDim.x >> 5); ++w) {
            if (w < warp) wpre += sh[w];
            tot += sh[w];
        }
        if (b < B) off[b] = carry + wpre + x - v;
        carry += tot;
        __syncthreads();
    }
    if (tid == 0) off[B] = carry;
}

// stable scatter: one warp walks its chunk in order; per-bucket running
// counters start at offsets[b] + (items of bucket b in earlier chunks).
__global__ void bsort_scatter_kernel(const uint32_t* __restrict__ keys, uint64_t n, uint32_t B, uint32_t chunk,
                                     uint32_t nch, uint32_t* counts, const uint32_t* __restrict__ offsets,
                                     uint32_t* __restrict__ perm, bool use_smem) {
    extern __shared__ uint32_t run[];
    const uint32_t j = blockIdx.y, ch = blockIdx.x, lane = threadIdx.x;
    uint32_t* row = counts + (uint64_t(j) * nch + ch) * B;
    const uint32_t* off = offsets + uint64_t(j) * (B + 1);
    uint32_t* ctr = use_smem ? run : row;
    for (uint32_t b = lane; b < B; b += 32) ctr[b] = off[b] + row[b];
    __syncwarp();
    const uint64_t lo = uint64_t(ch) * chunk, hi = min_u64(n, lo + chunk);
    const uint32_t* kk = keys + uint64_t(j) * n;
    uint32_t* pp = perm + uint64_t(j) * n;
    for (uint64_t i0 = lo; i0 < hi; i0 += 32) {
        const uint64_t i = i0 + lane;
        const bool ok = i < hi;
        const uint32_t key = ok ? kk[i] : 0xffffffffu;
        const uint32_t peers = __match_any_sync(kFull, key);
        const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
        const uint32_t base = ok ? ctr[key] : 0u;
        __syncwarp();
        if (ok) {
            pp[base + rank] = static_cast<uint32_t>(i);
            if (rank == 0) ctr[key] = base + __popc(peers);
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------------- update
// sums[c][t] = serial fold over cluster c's points in id order (kmeans.cpp:155-161),
// centroid = float(sum * (1 / count)) (kmeans.cpp:163-168); empty clusters untouched.
__global__ void update_kernel(const float* __restrict__ proj, const KJob* __restrict__ jobs, uint64_t n, uint32_t k,
                              const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ perm, float* cent) {
    const uint32_t j = blockIdx.y;
    const KJob jb = jobs[j];
    const uint32_t h = jb.h;
    const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (t >= uint64_t(k) * h) return;
    const uint32_t c = static_cast<uint32_t>(t / h), dim = static_cast<uint32_t>(t % h);
    const uint32_t* off = offsets + uint64_t(j) * (k + 1);
    const uint32_t b = off[c], e = off[c + 1];
    if (b == e) return;
    const uint32_t* pp = perm + uint64_t(j) * n;
    const float* x = proj + jb.off + dim;
    double sum = 0.0;
    uint32_t p = b;
    for (; p + 8 <= e; p += 8) {
        uint32_t id[8];
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) id[u] = __ldg(pp + p + u);
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldg(x + uint64_t(id[u]) * h);
#pragma unroll
        for (int u = 0; u < 8; ++u) sum = __dadd_rn(sum, static_cast<double>(v[u]));
    }
    for (; p < e; ++p) sum = __dadd_rn(sum, static_cast<double>(__ldg(x + uint64_t(__ldg(pp + p)) * h)));
    const double inv = 1.0 / static_cast<double>(e - b);
    cent[jb.coff + uint64_t(c) * h + dim] = __double2float_rn(__dmul_rn(sum, inv));
}

// The same sums folded exactly in parallel: one CTA per (job, cluster, dim). A signed running sum
// s with |s| in [2^e, 2^(e+1)) moves in steps of U = ulp(s): while every partial sum keeps s's sign
// and binade, fl(s + a) = s + U rint(a / U) (ties excepted), so a tile is an int64 block scan of
// rint(a_i / U) up to its first element that leaves the binade (up or down), is a tie, or meets a
// zero / subnormal s; that element gets one serial __dadd_rn and the scan resumes. Measured at cfg4
// (16 jobs x 64 clusters x 6 dims, 10M points): 50 ms per Lloyd round with one thread per column.
template <class F>
__device__ double fold_signed(F load, uint32_t count) {
    __shared__ long long wsum[8];
    __shared__ uint32_t s_bad;
    __shared__ double s_run;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    constexpr long long kTwo52 = 4503599627370496ll, kTwo53 = 9007199254740992ll;
    if (tid == 0) s_run = 0.0;
    __syncthreads();
    for (uint32_t base = 0; base < count; base += 2048) {
        const uint32_t len = min(2048u, count - base);
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t i = tid * 8 + u;
            v[u] = i < len ? load(base + i) : 0.0;
        }
        uint32_t start = 0;
        while (start < len) {
            const double s0 = s_run;  // exact running sum before element `start`
            const bool tiny = !(fabs(s0) >= 2.2250738585072014e-308);  // 0 or subnormal
            const double U = tiny ? 0.0 : ldexp(1.0, ilogb(s0) - 52);
            const long long S0 = tiny ? 0 : static_cast<long long>(s0 / U);  // exact, |S0| in [2^52, 2^53)
            long long r[8];
            bool badv[8];
            long long loc = 0;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t i = tid * 8 + u;
                const bool live = i >= start && i < len;
                r[u] = 0;
                badv[u] = false;
                if (live) {
                    if (tiny) {
                        badv[u] = v[u] != 0.0;
                    } else {
                        const double q = v[u] / U;  // exact (power-of-two scaling) unless huge
                        if (!(fabs(q) < 4503599627370496.0)) {
                            badv[u] = true;
                        } else {
                            const double m = floor(q);
                            const double f = q - m;  // exact
                            badv[u] = f == 0.5;  // a rounding tie: the result depends on s's last bit
                            r[u] = static_cast<long long>(f > 0.5 ? m + 1.0 : m);
                        }
                    }
                }
                if (badv[u]) r[u] = 0;
                loc += r[u];
            }
            long long x = loc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const long long y = __shfl_up_sync(kFull, x, o);
                if (lane >= static_cast<uint32_t>(o)) x += y;
            }
            if (lane == 31) wsum[warp] = x;
            if (tid == 0) s_bad = 0xffffffffu;
            __syncthreads();
            long long wpre = 0, tot = 0;
            for (uint32_t w = 0; w < 8; ++w) {
                if (w < warp) wpre += wsum[w];
                tot += wsum[w];
            }
            long long run = wpre + (x - loc);
            uint32_t first_bad = 0xffffffffu;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t i = tid * 8 + u;
                if (i >= start && i < len && first_bad == 0xffffffffu) {
                    const long long t = S0 + run + r[u];  // the partial after this element, in units of U
                    const long long at = t < 0 ? -t : t;
                    if (badv[u] || (!tiny && ((t < 0) != (S0 < 0) || at < kTwo52 || at >= kTwo53))) first_bad = i;
                    run += r[u];
                }
            }
            if (first_bad != 0xffffffffu) atomicMin(&s_bad, first_bad);
            __syncthreads();
            const uint32_t bad = s_bad;
            if (bad == 0xffffffffu || bad >= len) {  // the whole rest of the tile stayed in the binade
                if (tid == 0) s_run = tiny ? s0 : __dmul_rn(static_cast<double>(S0 + tot), U);
                __syncthreads();
                break;
            }
            if (tid == (bad >> 3)) {  // its predecessor's exact value, then one serial add
                long long rb = wpre + (x - loc);
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    if (tid * 8 + u < bad && tid * 8 + u >= start) rb += r[u];
                }
                const double prev = tiny ? s0 : __dmul_rn(static_cast<double>(S0 + rb), U);
                s_run = __dadd_rn(prev, v[bad & 7u]);
            }
            __syncthreads();
            start = bad + 1;
        }
    }
    const double out = s_run;
    __syncthreads();
    return out;
}

__global__ void __launch_bounds__(256) update_fold_kernel(const float* __restrict__ proj, const KJob* __restrict__ jobs,
                                                          uint64_t n, uint32_t k, const uint32_t* __restrict__ offsets,
                                                          const uint32_t* __restrict__ perm, float* cent) {
    const uint32_t j = blockIdx.y;
    const KJob jb = jobs[j];
    const uint32_t h = jb.h;
    const uint32_t c = blockIdx.x / h, dim = blockIdx.x % h;
    if (c >= k) return;
    const uint32_t* off = offsets + uint64_t(j) * (k + 1);
    const uint32_t b = off[c], e = off[c + 1];
    if (b == e) return;  // empty: repaired by the caller
    const uint32_t* pp = perm + uint64_t(j) * n + b;
    const float* x = proj + jb.off + dim;
    const double sum = fold_signed([&](uint32_t i) { return static_cast<double>(__ldg(x + uint64_t(__ldg(pp + i)) * h)); },
                                   e - b);
    if (threadIdx.x == 0) {
        const double inv = 1.0 / static_cast<double>(e - b);
        cent[jb.coff + uint64_t(c) * h + dim] = __double2float_rn(__dmul_rn(sum, inv));
    }
}

// ------------------------------------------------------------------- repair
struct FarArgs {
    uint32_t job, cluster;
};

// farthest point from the stale centroid, strict '>' => lowest id on ties
__global__ void farthest_partial_kernel(const float* __restrict__ proj, const KJob* __restrict__ jobs, uint64_t n,
                                        const float* __restrict__ cent, FarArgs fa, double* pd, uint32_t* pi) {
    __shared__ double sd[8];
    __shared__ uint32_t si[8];
    const KJob jb = jobs[fa.job];
    const float* stale = cent + jb.coff + uint64_t(fa.cluster) * jb.h;
    const float* x = proj + jb.off;
    double bd = -1.0;
    uint32_t bi = 0xffffffffu;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const double dist = sqdist4(x + i * jb.h, stale, jb.h);
        if (dist > bd) {
            bd = dist;
            bi = static_cast<uint32_t>(i);
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double od = __shfl_xor_sync(kFull, bd, o);
        const uint32_t oi = __shfl_xor_sync(kFull, bi, o);
        if (od > bd || (od == bd && oi < bi)) {
            bd = od;
            bi = oi;
        }
    }
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        sd[warp] = bd;
        si[warp] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w) {
            if (sd[w] > bd || (sd[w] == bd && si[w] < bi)) {
                bd = sd[w];
                bi = si[w];
            }
        }
        pd[blockIdx.x] = bd;
        pi[blockIdx.x] = bi;
    }
}

__global__ void farthest_final_kernel(const float* proj, const KJob* jobs, FarArgs fa, const double* pd,
                                      const uint32_t* pi, uint32_t parts, float* cent) {
    __shared__ uint32_t far;
    if (threadIdx.x == 0) {
        double bd = -1.0;
        uint32_t bi = 0xffffffffu;
        for (uint32_t b = 0; b < parts; ++b) {
            if (pd[b] > bd || (pd[b] == bd && pi[b] < bi)) {
                bd = pd[b];
                bi = pi[b];
            }
        }
        far = bi;
    }
    __syncthreads();
    const KJob jb = jobs[fa.job];
    for (uint32_t t = threadIdx.x; t < jb.h; t += blockDim.x) {
        cent[jb.coff + uint64_t(fa.cluster) * jb.h + t] = proj[jb.off + uint64_t(far) * jb.h + t];
    }
}

// ---------------------------------------------------------------------- IMI
__global__ void cell_keys_kernel(const uint32_t* __restrict__ assign, uint64_t n, uint32_t k, uint32_t ns,
                                 uint32_t* __restrict__ keys) {
    const uint32_t s = blockIdx.y;
    const uint32_t* a1 = assign + uint64_t(2 * s) * n;
    const uint32_t* a2 = assign + uint64_t(2 * s + 1) * n;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        keys[uint64_t(s) * n + i] = a1[i] * k + a2[i];
    }
}

// ==================================================================== host
unsigned grid_for(uint64_t n, unsigned per = 256, unsigned cap = 148 * 8) {
    const uint64_t b = (n + per - 1) / per;
    return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(b, cap)));
}

// Stable bucket sort of J problems (keys < B) -> offsets J x (B+1), perm J x n.
void bucket_sort(const uint32_t* keys, uint64_t n, uint32_t B, uint32_t J, uint32_t* offsets, uint32_t* perm,
                 cudaStream_t st) {
    uint64_t chunk = 2048;
    const uint64_t budget = 16ull << 20;  // count-matrix entries per problem
    if ((n + chunk - 1) / chunk * B > budget) chunk = ((n * B + budget - 1) / budget + 31) / 32 * 32;
    const uint32_t nch = static_cast<uint32_t>((n + chunk - 1) / chunk);
    const bool use_smem = uint64_t(B) * 4 <= 48 * 1024;
    Dev<uint32_t> counts(uint64_t(J) * nch * B), totals(uint64_t(J) * B);
    if (!use_smem) BCUDA(cudaMemsetAsync(counts.p, 0, counts.n * 4, st));
    const dim3 g(nch, J);
    bsort_hist_kernel<<<g, 256, use_smem ? B * 4 : 0, st>>>(keys, n, B, static_cast<uint32_t>(chunk), nch, counts.p,
                                                            use_smem);
    BCUDA(cudaGetLastError());
    bsort_colscan_kernel<<<grid_for(uint64_t(J) * B, 256, 1u << 30), 256, 0, st>>>(counts.p, B, nch, J, totals.p);
    BCUDA(cudaGetLastError());
    bsort_offsets_kernel<<<J, 1024, 0, st>>>(totals.p, B, offsets);
    BCUDA(cudaGetLastError());
    bsort_scatter_kernel<<<g, 32, use_smem ? B * 4 : 0, st>>>(keys, n, B, static_cast<uint32_t>(chunk), nch, counts.p,
                                                            offsets, perm, use_smem);
    BCUDA(cudaGetLastError());
    BCUDA(cudaStreamSynchronize(st));
}

void launch_assign(const float* proj, const KJob* jobs, uint64_t n, uint32_t k, uint32_t hmax, const float* cent,
                   uint32_t* assign, uint32_t J, cudaStream_t st) {
    const size_t smem = size_t(k) * hmax * (hmax <= 32 ? 8 + 4 : 8);  // doubles (+ the fp32 screen's floats)
    if (smem > 200 * 1024) raise(SUCO_ERR_INTERNAL, "k x h centroid table exceeds shared memory");
    const dim3 g(grid_for(n, 256, 148 * 4), J);
    auto go = [&](auto kern) {
        if (smem > 48 * 1024) BCUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        kern<<<g, 256, smem, st>>>(proj, jobs, n, k, cent, assign);
        BCUDA(cudaGetLastError());
    };
    if (hmax <= 8) go(assign_kernel<8>);
    else if (hmax <= 16) go(assign_kernel<16>);
    else if (hmax <= 32) go(assign_kernel<32>);
    else go(assign_kernel<0>);
}

// The whole k-means of J jobs sharing n and k (kmeans.cpp:118-194).
// proj/jobs/cent are device arrays; host_jobs mirrors jobs; seeds per job.
void kmeans_jobs(const float* proj, const std::vector<KJob>& host_jobs, const KJob* jobs, uint64_t n, uint32_t k,
                 uint32_t iterations, const std::vector<uint64_t>& seeds, float* cent, uint32_t* assign,
                 std::vector<std::vector<uint32_t>>* repaired, cudaStream_t st, bool kpp_serial) {
    const uint32_t J = static_cast<uint32_t>(host_jobs.size());
    uint32_t hmax = 0;
    for (const KJob& jb : host_jobs) hmax = std::max(hmax, jb.h);

    // integer certificate per job: integer values with n * h * (2 max|v|)^2 < 2^52
    Dev<unsigned int> nonint(J), maxbits(J);
    BCUDA(cudaMemsetAsync(nonint.p, 0, J * 4, st));
    BCUDA(cudaMemsetAsync(maxbits.p, 0, J * 4, st));
    int_check_kernel<<<dim3(grid_for(n * hmax, 256, 148 * 4), J), 256, 0, st>>>(proj, jobs, n, nonint.p, maxbits.p);
    BCUDA(cudaGetLastError());
    std::vector<unsigned int> hn(J), hm(J);
    BCUDA(cudaMemcpyAsync(hn.data(), nonint.p, J * 4, cudaMemcpyDeviceToHost, st));
    BCUDA(cudaMemcpyAsync(hm.data(), maxbits.p, J * 4, cudaMemcpyDeviceToHost, st));
    BCUDA(cudaStreamSynchronize(st));
    std::vector<uint8_t> exact(J);
    for (uint32_t j = 0; j < J; ++j) {
        float mx;
        std::memcpy(&mx, &hm[j], 4);
        const double span = 2.0 * double(mx);
        exact[j] = (hn[j] == 0) && (double(n) * host_jobs[j].h * span * span < 4503599627370496.0);  // 2^52
    }

    // host replay of each job's RNG stream: first pick, then k-1 uniforms
    std::vector<uint32_t> pick0(J);
    std::vector<double> unis(uint64_t(J) * std::max<uint32_t>(k, 1));
    for (uint32_t j = 0; j < J; ++j) {
        Mt64 g(seeds[j]);
        pick0[j] = static_cast<uint32_t>(g.uniform_below(n));
        for (uint32_t c = 0; c + 1 < k; ++c) unis[uint64_t(j) * k + c] = g.uniform_unit();
    }
    Dev<double> min_dist(uint64_t(J) * n), prefix(kpp_serial ? uint64_t(J) * n : 1), d_unis(unis.size());
    Dev<uint8_t> chosen(uint64_t(J) * n), d_exact(J);
    Dev<uint32_t> pick(J), used(J);
    BCUDA(cudaMemcpyAsync(d_unis.p, unis.data(), unis.size() * 8, cudaMemcpyHostToDevice, st));
    BCUDA(cudaMemcpyAsync(d_exact.p, exact.data(), J, cudaMemcpyHostToDevice, st));
    BCUDA(cudaMemcpyAsync(pick.p, pick0.data(), J * 4, cudaMemcpyHostToDevice, st));
    BCUDA(cudaMemsetAsync(used.p, 0, J * 4, st));
    kpp_init_kernel<<<grid_for(n * J), 256, 0, st>>>(min_dist.p, chosen.p, n, J);
    copy_centroid_kernel<<<J, 64, 0, st>>>(proj, jobs, pick.p, 0, cent);
    BCUDA(cudaGetLastError());
    const dim3 gu(grid_for(n, 256, 148 * 4), J);
    // the chunked fold (kpp_chunk_*); SUCO_KPP_SERIAL keeps the one-CTA-per-job kernel for A/B
    const uint32_t NC = static_cast<uint32_t>((n + kKppChunk - 1) / kKppChunk);
    Dev<double> csum(uint64_t(J) * NC), csin(uint64_t(J) * NC), csout(uint64_t(J) * NC);
    Dev<uint32_t> cready(uint64_t(J) * NC), ticket(k);
    BCUDA(cudaMemsetAsync(cready.p, 0, uint64_t(J) * NC * 4, st));
    BCUDA(cudaMemsetAsync(ticket.p, 0, uint64_t(k) * 4, st));
    for (uint32_t c = 1; c < k; ++c) {
        kpp_update_kernel<<<gu, 256, 0, st>>>(proj, jobs, n, pick.p, min_dist.p, chosen.p);
        if (kpp_serial) {
            kpp_select_kernel<<<J, 256, 0, st>>>(proj, jobs, n, c, min_dist.p, chosen.p, d_exact.p, d_unis.p, k,
                                                 used.p, pick.p, prefix.p, cent, kpp_serial);
        } else {
            kpp_chunk_sum_kernel<<<dim3(NC, J), 256, 0, st>>>(min_dist.p, n, NC, csum.p);
            kpp_chunk_fold_kernel<<<NC * J, 256, 0, st>>>(min_dist.p, n, NC, J, d_exact.p, csum.p, csin.p, csout.p,
                                                          cready.p, ticket.p + c, c);
            kpp_pick_kernel<<<J, 256, 0, st>>>(proj, jobs, n, c, min_dist.p, chosen.p, d_exact.p, d_unis.p, k, used.p,
                                               pick.p, csin.p, csout.p, NC, cent);
        }
        BCUDA(cudaGetLastError());
    }
    min_dist.release();
    prefix.release();
    chosen.release();

    // Lloyd rounds
    Dev<uint32_t> offsets(uint64_t(J) * (k + 1)), perm(uint64_t(J) * n);
    std::vector<uint32_t> hoff(uint64_t(J) * (k + 1));
    Dev<double> pd(148 * 4);
    Dev<uint32_t> pi(148 * 4);
    const unsigned fparts = grid_for(n, 256, 148 * 4);
    for (uint32_t it = 0; it < iterations; ++it) {
        launch_assign(proj, jobs, n, k, hmax, cent, assign, J, st);
        bucket_sort(assign, n, k, J, offsets.p, perm.p, st);
        if (kpp_serial) {  // (A/B and tests: the one-thread-per-column fold)
            update_kernel<<<dim3(grid_for(uint64_t(k) * hmax, 128, 1u << 30), J), 128, 0, st>>>(proj, jobs, n, k,
                                                                                               offsets.p, perm.p, cent);
        } else {
            update_fold_kernel<<<dim3(k * hmax, J), 256, 0, st>>>(proj, jobs, n, k, offsets.p, perm.p, cent);
        }
        BCUDA(cudaGetLastError());
        BCUDA(cudaMemcpyAsync(hoff.data(), offsets.p, hoff.size() * 4, cudaMemcpyDeviceToHost, st));
        BCUDA(cudaStreamSynchronize(st));
        for (uint32_t j = 0; j < J; ++j) {
            for (uint32_t c = 0; c < k; ++c) {
                if (hoff[uint64_t(j) * (k + 1) + c + 1] != hoff[uint64_t(j) * (k + 1) + c]) continue;
                const FarArgs fa{j, c};
                farthest_partial_kernel<<<fparts, 256, 0, st>>>(proj, jobs, n, cent, fa, pd.p, pi.p);
                farthest_final_kernel<<<1, 64, 0, st>>>(proj, jobs, fa, pd.p, pi.p, fparts, cent);
                BCUDA(cudaGetLastError());
                if (repaired) (*repaired)[j].push_back(c);
            }
        }
    }
    launch_assign(proj, jobs, n, k, hmax, cent, assign, J, st);
    BCUDA(cudaStreamSynchronize(st));
}

}  // namespace

// The 2*N_s jobs' KJob table for `rows` points (job-major projections, rows x h each).
static uint64_t job_table(const HostLayout& L, uint32_t k, uint64_t rows, std::vector<KJob>& hj,
                          std::vector<uint32_t>& dim_off, std::vector<uint32_t>& dims, uint64_t* coff_out) {
    const uint32_t ns = L.ns, J = 2 * ns;
    hj.assign(J, KJob{});
    dim_off.assign(J + 1, 0);
    dims.clear();
    uint64_t off = 0, coff = 0;
    uint32_t pos = 0;
    for (uint32_t s = 0; s < ns; ++s) {
        for (uint32_t half = 0; half < 2; ++half) {
            const uint32_t j = 2 * s + half;
            const uint32_t h = half == 0 ? L.h1(s) : L.h2(s);
            hj[j] = KJob{h, 0, off, coff};
            off += rows * h;
            coff += uint64_t(k) * h;
            dim_off[j] = static_cast<uint32_t>(dims.size());
            const uint32_t b = pos + (half == 0 ? 0 : L.split[s]);
            for (uint32_t t = 0; t < h; ++t) dims.push_back(L.dims[b + t]);
        }
        pos += L.sizes[s];
    }
    dim_off[J] = static_cast<uint32_t>(dims.size());
    *coff_out = coff;
    return off;
}

// Every row to its nearest centroid of each job (kmeans.cpp:19-33, the final-pass rule), in row
// chunks: project the chunk, assign it, scatter its J columns into assign (J x n).
static void assign_rows(const float* d_data, uint64_t n, uint32_t d, const HostLayout& L, uint32_t k,
                        const std::vector<KJob>& hj, const uint32_t* ddims, const uint32_t* ddoff, const float* cent,
                        uint32_t* assign, cudaStream_t st, uint64_t chunk_rows) {
    const uint32_t J = 2 * L.ns;
    uint32_t hmax = 0;
    for (const KJob& jb : hj) hmax = std::max(hmax, jb.h);
    uint64_t chunk = std::max<uint64_t>(1, (2ull << 30) / (uint64_t(d) * 4));  // 2 GB of projections
    if (chunk_rows) chunk = chunk_rows;  // tests
    chunk = std::max<uint64_t>(1, std::min<uint64_t>(n, chunk));
    std::vector<KJob> cj;
    std::vector<uint32_t> cdo, cdims;
    uint64_t ccoff = 0;
    const uint64_t coffs = job_table(L, k, chunk, cj, cdo, cdims, &ccoff);
    Dev<KJob> cjobs(J);
    Dev<float> cproj(coffs);
    Dev<uint32_t> cassign(uint64_t(J) * chunk);
    // the centroid offsets of `hj` (any row count) and `cj` agree: both follow the job order
    BCUDA(cudaMemcpyAsync(cjobs.p, cj.data(), J * sizeof(KJob), cudaMemcpyHostToDevice, st));
    for (uint64_t r0 = 0; r0 < n; r0 += chunk) {
        const uint64_t nc = std::min(chunk, n - r0);
        project_kernel<<<dim3(grid_for(nc, 256, 148 * 4), J), 256, 0, st>>>(d_data + r0 * d, nc, d, ddims, ddoff,
                                                                            cjobs.p, cproj.p, nullptr);
        BCUDA(cudaGetLastError());
        launch_assign(cproj.p, cjobs.p, nc, k, hmax, cent, cassign.p, J, st);
        BCUDA(cudaMemcpy2DAsync(assign + r0, n * 4, cassign.p, nc * 4, nc * 4, J, cudaMemcpyDeviceToDevice, st));
    }
    BCUDA(cudaStreamSynchronize(st));
}

void build_index_device(const float* d_data, uint64_t n, uint32_t d, const HostLayout& L, const suco_index_params& p,
                        BuildOutputs& out, cudaStream_t st, const Tuning& tune, const uint32_t* train,
                        uint64_t n_train) {
    const uint32_t ns = L.ns, J = 2 * ns, k = p.k_half;
    // k-means fits on every row, or (sampled build) on the training rows only
    const uint64_t nfit = train ? n_train : n;
    std::vector<KJob> hj;
    std::vector<uint32_t> dim_off, dims;
    uint64_t coff = 0;
    const uint64_t off = job_table(L, k, nfit, hj, dim_off, dims, &coff);
    Dev<KJob> jobs(J);
    Dev<uint32_t> ddims(dims.size()), ddoff(J + 1), dtrain(train ? n_train : 1);
    Dev<float> proj(off), cent(coff);
    BCUDA(cudaMemcpyAsync(jobs.p, hj.data(), J * sizeof(KJob), cudaMemcpyHostToDevice, st));
    BCUDA(cudaMemcpyAsync(ddims.p, dims.data(), dims.size() * 4, cudaMemcpyHostToDevice, st));
    BCUDA(cudaMemcpyAsync(ddoff.p, dim_off.data(), (J + 1) * 4, cudaMemcpyHostToDevice, st));
    if (train) BCUDA(cudaMemcpyAsync(dtrain.p, train, n_train * 4, cudaMemcpyHostToDevice, st));
    project_kernel<<<dim3(grid_for(nfit, 256, 148 * 4), J), 256, 0, st>>>(d_data, nfit, d, ddims.p, ddoff.p, jobs.p,
                                                                          proj.p, train ? dtrain.p : nullptr);
    BCUDA(cudaGetLastError());

    std::vector<uint64_t> seeds(J);
    for (uint32_t j = 0; j < J; ++j) seeds[j] = derive_seed(p.seed, j);  // index.cpp:131
    Dev<uint32_t> assign(uint64_t(J) * n);
    {
        Dev<uint32_t> fit_assign(train ? uint64_t(J) * n_train : 1);
        kmeans_jobs(proj.p, hj, jobs.p, nfit, k, p.iterations, seeds, cent.p, train ? fit_assign.p : assign.p, nullptr,
                    st, tune.kpp_serial);
    }
    proj.release();
    dtrain.release();
    if (train) assign_rows(d_data, n, d, L, k, hj, ddims.p, ddoff.p, cent.p, assign.p, st, tune.build_chunk);

    // centroids to the host (tiny)
    std::vector<float> hc(coff);
    BCUDA(cudaMemcpyAsync(hc.data(), cent.p, coff * 4, cudaMemcpyDeviceToHost, st));
    BCUDA(cudaStreamSynchronize(st));
    out.cent1->assign(ns, {});
    out.cent2->assign(ns, {});
    for (uint32_t s = 0; s < ns; ++s) {
        const KJob& a = hj[2 * s];
        const KJob& b = hj[2 * s + 1];
        (*out.cent1)[s].assign(hc.begin() + a.coff, hc.begin() + a.coff + uint64_t(k) * a.h);
        (*out.cent2)[s].assign(hc.begin() + b.coff, hc.begin() + b.coff + uint64_t(k) * b.h);
    }

    // IMI per subspace: stable counting sort by c1 * k + c2 (index.cpp:69-96)
    Dev<uint32_t> keys(uint64_t(ns) * n);
    cell_keys_kernel<<<dim3(grid_for(n, 256, 148 * 4), ns), 256, 0, st>>>(assign.p, n, k, ns, keys.p);
    BCUDA(cudaGetLastError());
    bucket_sort(keys.p, n, k * k, ns, out.cell_off, out.ids, st);
}

void build_shard_device(const float* d_rows, uint64_t n_local, uint64_t n_global, uint32_t d, uint32_t b,
                        const HostLayout& L, const suco_index_params& p, suco_comm* comm, BuildOutputs& out,
                        uint32_t* cell_size, cudaStream_t st, const Tuning& tune, const uint32_t* train,
                        uint64_t n_train) {
    const uint32_t ns = L.ns, J = 2 * ns, k = p.k_half;
    const uint32_t G = static_cast<uint32_t>(comm->size), me = static_cast<uint32_t>(comm->rank);
    const uint64_t nfit = train ? n_train : n_global;
    auto owner_of = [&](uint64_t g) { return static_cast<uint32_t>((g / b) % G); };
    auto local_of = [&](uint64_t g) { return ((g / b) / G) * b + g % b; };
    // the training rows in global id order: which rank holds each and where in that rank's list
    std::vector<uint64_t> cnt(G, 0);
    std::vector<uint32_t> src(nfit);       // rank-major gathered position of training row t
    std::vector<uint32_t> mine;            // this rank's training rows (local ids), id order
    for (uint64_t t = 0; t < nfit; ++t) {
        const uint64_t g = train ? train[t] : t;
        const uint32_t r = owner_of(g);
        src[t] = static_cast<uint32_t>(cnt[r]++);  // rank offset added below, once maxcnt is known
        if (r == me) mine.push_back(static_cast<uint32_t>(local_of(g)));
    }
    uint64_t maxcnt = 1;
    for (uint64_t c : cnt) maxcnt = std::max(maxcnt, c);
    for (uint64_t t = 0; t < nfit; ++t) {
        const uint64_t g = train ? train[t] : t;
        src[t] = static_cast<uint32_t>(uint64_t(owner_of(g)) * maxcnt + src[t]);
    }
    if (uint64_t(G) * maxcnt > 0xFFFFFFFFull) raise(SUCO_ERR_CONTRACT, "sharded build: training rows exceed 32-bit ids");

    // 1. project this rank's training rows for every job (job-major, maxcnt rows per job)
    std::vector<KJob> hj;
    std::vector<uint32_t> dim_off, dims;
    uint64_t coff = 0;
    const uint64_t off = job_table(L, k, maxcnt, hj, dim_off, dims, &coff);
    Dev<KJob> jobs(J);
    Dev<uint32_t> ddims(dims.size()), ddoff(J + 1), drows(mine.size());
    Dev<float> proj(off), cent(coff);
    BCUDA(cudaMemcpyAsync(jobs.p, hj.data(), J * sizeof(KJob), cudaMemcpyHostToDevice, st));
    BCUDA(cudaMemcpyAsync(ddims.p, dims.data(), dims.size() * 4, cudaMemcpyHostToDevice, st));
    BCUDA(cudaMemcpyAsync(ddoff.p, dim_off.data(), (J + 1) * 4, cudaMemcpyHostToDevice, st));
    if (!mine.empty()) {
        BCUDA(cudaMemcpyAsync(drows.p, mine.data(), mine.size() * 4, cudaMemcpyHostToDevice, st));
        project_kernel<<<dim3(grid_for(mine.size(), 256, 148 * 4), J), 256, 0, st>>>(
            d_rows, mine.size(), d, ddims.p, ddoff.p, jobs.p, proj.p, drows.p);
        BCUDA(cudaGetLastError());
    }

    // 2. job j's column gathers on rank j % G, in global training order (the k-means input order)
    std::vector<uint32_t> own_jobs;
    for (uint32_t j = 0; j < J; ++j) {
        if (j % G == me) own_jobs.push_back(j);
    }
    const uint32_t Jr = static_cast<uint32_t>(own_jobs.size());
    std::vector<KJob> hjr(Jr);
    uint64_t roff = 0, rcoff = 0;
    uint32_t hmax = 1;
    for (uint32_t i = 0; i < Jr; ++i) {
        const uint32_t h = hj[own_jobs[i]].h;
        hjr[i] = KJob{h, 0, roff, rcoff};
        roff += nfit * h;
        rcoff += uint64_t(k) * h;
        hmax = std::max(hmax, h);
    }
    Dev<float> fit(Jr ? roff : 1), gathered(Jr ? uint64_t(G) * maxcnt * hmax : 1), rcent(Jr ? rcoff : 1);
    Dev<uint32_t> dsrc(Jr ? nfit : 1);
    if (Jr) BCUDA(cudaMemcpyAsync(dsrc.p, src.data(), nfit * 4, cudaMemcpyHostToDevice, st));
    for (uint32_t j = 0; j < J; ++j) {
        const int root = static_cast<int>(j % G);
        comm->gather(proj.p + hj[j].off, gathered.p, maxcnt * hj[j].h * 4, root, st);
        if (root == static_cast<int>(me)) {
            const uint32_t i = static_cast<uint32_t>(std::find(own_jobs.begin(), own_jobs.end(), j) - own_jobs.begin());
            gather_rows_kernel<<<grid_for(nfit * hj[j].h), 256, 0, st>>>(gathered.p, dsrc.p, nfit, hj[j].h,
                                                                       fit.p + hjr[i].off);
            BCUDA(cudaGetLastError());
        }
    }
    proj.release();
    gathered.release();
    dsrc.release();

    // 3. the owned k-means jobs (seeds derive_seed(seed, j), index.cpp:131), then every job's
    //    centroids broadcast from its owner
    if (Jr) {
        std::vector<uint64_t> seeds(Jr);
        for (uint32_t i = 0; i < Jr; ++i) seeds[i] = derive_seed(p.seed, own_jobs[i]);
        Dev<KJob> rjobs(Jr);
        Dev<uint32_t> rassign(uint64_t(Jr) * nfit);
        BCUDA(cudaMemcpyAsync(rjobs.p, hjr.data(), Jr * sizeof(KJob), cudaMemcpyHostToDevice, st));
        kmeans_jobs(fit.p, hjr, rjobs.p, nfit, k, p.iterations, seeds, rcent.p, rassign.p, nullptr, st, tune.kpp_serial);
        for (uint32_t i = 0; i < Jr; ++i) {
            BCUDA(cudaMemcpyAsync(cent.p + hj[own_jobs[i]].coff, rcent.p + hjr[i].coff, uint64_t(k) * hjr[i].h * 4,
                                  cudaMemcpyDeviceToDevice, st));
        }
    }
    fit.release();
    for (uint32_t j = 0; j < J; ++j) comm->broadcast(cent.p + hj[j].coff, uint64_t(k) * hj[j].h * 4, int(j % G), st);

    // 4. every local row to its nearest centroid; the local IMI (local ids, ascending per cell)
    Dev<uint32_t> assign(uint64_t(J) * std::max<uint64_t>(n_local, 1));
    if (n_local) assign_rows(d_rows, n_local, d, L, k, hj, ddims.p, ddoff.p, cent.p, assign.p, st, tune.build_chunk);
    std::vector<float> hc(coff);
    BCUDA(cudaMemcpyAsync(hc.data(), cent.p, coff * 4, cudaMemcpyDeviceToHost, st));
    BCUDA(cudaStreamSynchronize(st));
    out.cent1->assign(ns, {});
    out.cent2->assign(ns, {});
    for (uint32_t s = 0; s < ns; ++s) {
        const KJob& a = hj[2 * s];
        const KJob& c = hj[2 * s + 1];
        (*out.cent1)[s].assign(hc.begin() + a.coff, hc.begin() + a.coff + uint64_t(k) * a.h);
        (*out.cent2)[s].assign(hc.begin() + c.coff, hc.begin() + c.coff + uint64_t(k) * c.h);
    }
    Dev<uint32_t> keys(uint64_t(ns) * std::max<uint64_t>(n_local, 1));
    cell_keys_kernel<<<dim3(grid_for(n_local, 256, 148 * 4), ns), 256, 0, st>>>(assign.p, n_local, k, ns, keys.p);
    BCUDA(cudaGetLastError());
    bucket_sort(keys.p, n_local, k * k, ns, out.cell_off, out.ids, st);

    // 5. global cell sizes (every shard's Dynamic-Activation cut is the global one)
    BCUDA(launch_cell_sizes(out.cell_off, ns, k * k, cell_size, st));
    comm->allreduce_sum_u32(cell_size, uint64_t(ns) * k * k, st);
    BCUDA(cudaStreamSynchronize(st));
}

void kmeans_device_host_io(const float* points, uint64_t n, uint32_t dim, uint32_t k, uint32_t iterations, uint64_t seed,
                           float* centroids, uint32_t* assignments, uint32_t* repaired, uint32_t* num_repaired) {
    cudaStream_t st = nullptr;
    BCUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{st};
    std::vector<KJob> hj{KJob{dim, 0, 0, 0}};
    Dev<KJob> jobs(1);
    Dev<float> proj(n * dim), cent(uint64_t(k) * dim);
    Dev<uint32_t> assign(n);
    BCUDA(cudaMemcpyAsync(jobs.p, hj.data(), sizeof(KJob), cudaMemcpyHostToDevice, st));
    BCUDA(cudaMemcpyAsync(proj.p, points, n * dim * 4, cudaMemcpyHostToDevice, st));
    std::vector<std::vector<uint32_t>> rep(1);
    kmeans_jobs(proj.p, hj, jobs.p, n, k, iterations, {seed}, cent.p, assign.p, &rep, st, tuning_from_env().kpp_serial);
    BCUDA(cudaMemcpyAsync(centroids, cent.p, uint64_t(k) * dim * 4, cudaMemcpyDeviceToHost, st));
    BCUDA(cudaMemcpyAsync(assignments, assign.p, n * 4, cudaMemcpyDeviceToHost, st));
    BCUDA(cudaStreamSynchronize(st));
    if (num_repaired) *num_repaired = static_cast<uint32_t>(rep[0].size());
    if (repaired) std::copy(rep[0].begin(), rep[0].end(), repaired);
}

void build_imi_host_io(const uint32_t* first, const uint32_t* second, uint64_t n, uint32_t k_half, uint64_t* offsets,
                       uint32_t* ids) {
    cudaStream_t st = nullptr;
    BCUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{st};
    const uint64_t K = uint64_t(k_half) * k_half;
    if (K > 0xFFFFFFFFull) raise(SUCO_ERR_CONTRACT, "build_imi: k_half^2 exceeds 32-bit cell ids");
    Dev<uint32_t> assign(2 * std::max<uint64_t>(n, 1)), keys(std::max<uint64_t>(n, 1)), off(K + 1), perm(std::max<uint64_t>(n, 1));
    if (n) {
        BCUDA(cudaMemcpyAsync(assign.p, first, n * 4, cudaMemcpyHostToDevice, st));
        BCUDA(cudaMemcpyAsync(assign.p + n, second, n * 4, cudaMemcpyHostToDevice, st));
        cell_keys_kernel<<<dim3(grid_for(n, 256, 148 * 4), 1), 256, 0, st>>>(assign.p, n, k_half, 1, keys.p);
        BCUDA(cudaGetLastError());
        bucket_sort(keys.p, n, static_cast<uint32_t>(K), 1, off.p, perm.p, st);
    } else {
        BCUDA(cudaMemsetAsync(off.p, 0, (K + 1) * 4, st));
    }
    std::vector<uint32_t> o32(K + 1);
    BCUDA(cudaMemcpyAsync(o32.data(), off.p, (K + 1) * 4, cudaMemcpyDeviceToHost, st));
    if (n) BCUDA(cudaMemcpyAsync(ids, perm.p, n * 4, cudaMemcpyDeviceToHost, st));
    BCUDA(cudaStreamSynchronize(st));
    for (uint64_t c = 0; c <= K; ++c) offsets[c] = o32[c];
}

}  // namespace suco_gpu
