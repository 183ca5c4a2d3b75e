// Small device utilities used while uploading/building an index.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "tuning.h"

namespace suco_gpu {
namespace {

__global__ void cell_sizes_kernel(const uint32_t* cell_off, uint32_t ns, uint32_t K, uint32_t* cell_size) {
    const uint64_t total = static_cast<uint64_t>(ns) * K;
    for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t s = t / K, c = t % K;
        const uint32_t* off = cell_off + s * (K + 1);
        cell_size[t] = off[c + 1] - off[c];
    }
}

// flag <- lowest index of a non-finite value (core.cpp:15-19 reports the index).
__global__ void check_finite_kernel(const float* data, uint64_t count, unsigned long long* first_bad) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t bits = __float_as_uint(data[i]);
        if ((bits & 0x7f800000u) == 0x7f800000u) atomicMin(first_bad, static_cast<unsigned long long>(i));
    }
}

// integer certificate: any non-integer value; largest |value| (as float bits)
// out[0] |= 1: some value is not an integer; out[1] = max |v| (float bits); out[2] |= 1: some v < 0.
__global__ void int_stats_kernel(const float* data, uint64_t count, unsigned int* out) {
    bool bad = false, neg = false;
    float mx = 0.f;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const float v = data[i];
        bad |= (v != truncf(v));
        neg |= (v < 0.f);
        mx = fmaxf(mx, fabsf(v));
    }
    bad = __any_sync(0xffffffffu, bad);
    neg = __any_sync(0xffffffffu, neg);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) {
        if (bad) atomicOr(out, 1u);
        atomicMax(out + 1, __float_as_uint(mx));
        if (neg) atomicOr(out + 2, 1u);
    }
}

// rows of u8-valued floats -> bytes, rows padded with zeros to dpad (a multiple of 16)
__global__ void pack_u8_kernel(const float* data, uint64_t n, uint32_t d, uint32_t dpad, uint8_t* out) {
    const uint64_t total = n * dpad;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t r = i / dpad;
        const uint32_t c = static_cast<uint32_t>(i % dpad);
        out[i] = c < d ? static_cast<uint8_t>(data[r * d + c]) : uint8_t(0);
    }
}

}  // namespace

// One warp per row: s = max|x| / 127, a = rint(x / s) in [-127, 127] (zero padding to qpad), and
// the row's bound terms (rerank_q8_kernel): |x|^2 (fp64 sum, rounded to f32), ||s a|| and
// ||x - s a|| (fp64, rounded up). A row whose terms are not finite gets s = -1: it always survives
// the screen.
// The int8 screen's records (rerank.cu). Plain (qpre = 0): [int8 row][meta = (s, |x|^2, ||s a|| up,
// ||e_x|| up)]. Prefix-bound layout (rerank_q8p_kernel): [meta0 = (s, |a_S|^2, ||e_x,S|| up, 0)]
// [dims 0 .. 16 qpre) in qsplit bytes, and [the other dims][meta1 = (|a|^2, ||e_x|| up, s, 0)] in
// qrec - qsplit bytes, S = the first 16 qpre dims. The two parts are two arrays: the n prefix parts
// back to back (stride qsplit: every candidate's first read — random accesses cost DRAM per access,
// not per byte (profiles/r02_gather_peak.json), so the dense array is what L2 and the DRAM pages
// see), then the n rests (stride qrec - qsplit, from byte n * qsplit). A row with a non-finite
// term gets s = -1 (always re-ranked exactly).
__global__ void pack_q8_kernel(const float* __restrict__ data, uint64_t n, uint32_t d, uint32_t qpad, uint32_t qrec,
                               uint32_t qpre, uint32_t qsplit, int8_t* __restrict__ out) {
    const uint32_t kPre = 16 * qpre;  // prefix dims
    const uint32_t lane = threadIdx.x & 31u;
    const bool split = qpre != 0;
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x / 32);
    for (uint64_t r = blockIdx.x * uint64_t(blockDim.x / 32) + (threadIdx.x >> 5); r < n; r += warps) {
        const float* x = data + r * d;
        int8_t* rec = out + r * qrec;                                  // plain records
        int8_t* recA = out + r * qsplit;                               // prefix part
        int8_t* recB = out + n * uint64_t(qsplit) + r * (qrec - qsplit);  // the rest
        float mx = 0.f;
        for (uint32_t i = lane; i < d; i += 32) mx = fmaxf(mx, fabsf(x[i]));
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const float s = mx / 127.f;
        double e2 = 0.0, a2 = 0.0, n2 = 0.0, e2s = 0.0, a2s = 0.0;
        for (uint32_t i = lane; i < qpad; i += 32) {
            float av = 0.f;
            if (i < d) {
                const float v = x[i];
                av = s > 0.f ? fminf(127.f, fmaxf(-127.f, rintf(v / s))) : 0.f;
                const double e = static_cast<double>(v) - static_cast<double>(s) * static_cast<double>(av);
                e2 += e * e;
                a2 += static_cast<double>(av) * static_cast<double>(av);
                n2 += static_cast<double>(v) * static_cast<double>(v);
                if (i < kPre) {
                    e2s += e * e;
                    a2s += static_cast<double>(av) * static_cast<double>(av);
                }
            }
            if (!split) rec[i] = static_cast<int8_t>(av);
            else if (i < kPre) recA[16 + i] = static_cast<int8_t>(av);
            else recB[i - kPre] = static_cast<int8_t>(av);
        }
        for (int o = 16; o > 0; o >>= 1) {
            e2 += __shfl_xor_sync(0xffffffffu, e2, o);
            a2 += __shfl_xor_sync(0xffffffffu, a2, o);
            n2 += __shfl_xor_sync(0xffffffffu, n2, o);
            e2s += __shfl_xor_sync(0xffffffffu, e2s, o);
            a2s += __shfl_xor_sync(0xffffffffu, a2s, o);
        }
        if (lane == 0) {
            const double A = static_cast<double>(s) * sqrt(a2) * (1.0 + 1e-12);
            const double R = sqrt(e2) * (1.0 + 1e-12);
            const double RS = sqrt(e2s) * (1.0 + 1e-12);
            const float fn2 = __double2float_rn(n2), fA = __double2float_ru(A), fR = __double2float_ru(R);
            const float fRS = __double2float_ru(RS);
            const bool ok = isfinite(fn2) && isfinite(fA) && isfinite(fR) && isfinite(fRS) && isfinite(s);
            const float fs = ok ? s : -1.f;
            if (!split) {
                *reinterpret_cast<float4*>(rec + qpad) = ok ? make_float4(s, fn2, fA, fR) : make_float4(-1.f, 0.f, 0.f, 0.f);
                for (uint32_t i = qpad + 16; i < qrec; ++i) rec[i] = 0;
            } else {
                for (uint32_t i = 16 + kPre; i < qsplit; ++i) recA[i] = 0;
                const uint32_t m1 = qpad - kPre;  // meta1 after the rest of the row
                *reinterpret_cast<uint4*>(recA) =
                    make_uint4(__float_as_uint(fs), static_cast<uint32_t>(a2s), __float_as_uint(fRS), 0u);
                *reinterpret_cast<uint4*>(recB + m1) =
                    make_uint4(static_cast<uint32_t>(a2), __float_as_uint(fR), __float_as_uint(fs), 0u);
                for (uint32_t i = m1 + 16; i < qrec - qsplit; ++i) recB[i] = 0;
            }
        }
    }
}

cudaError_t launch_pack_q8(const float* data, uint64_t n, uint32_t d, uint32_t qpad, uint32_t qrec, uint32_t qpre,
                           uint32_t qsplit, int8_t* out, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const uint64_t blocks = min_u64((n + 7) / 8, 148ull * 16);
    pack_q8_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(data, n, d, qpad, qrec, qpre, qsplit, out);
    return cudaGetLastError();
}

cudaError_t launch_pack_u8(const float* data, uint64_t n, uint32_t d, uint32_t dpad, uint8_t* out, cudaStream_t st) {
    const uint64_t blocks = min_u64((n * dpad + 255) / 256, 148ull * 16);
    pack_u8_kernel<<<static_cast<unsigned>(blocks ? blocks : 1), 256, 0, st>>>(data, n, d, dpad, out);
    return cudaGetLastError();
}

cudaError_t launch_int_stats(const float* data, uint64_t count, unsigned int* out2, cudaStream_t st) {
    const uint64_t blocks = min_u64((count + 255) / 256, 148ull * 16);
    int_stats_kernel<<<static_cast<unsigned>(blocks ? blocks : 1), 256, 0, st>>>(data, count, out2);
    return cudaGetLastError();
}

cudaError_t launch_cell_sizes(const uint32_t* cell_off, uint32_t ns, uint32_t K, uint32_t* cell_size, cudaStream_t st) {
    const uint64_t total = static_cast<uint64_t>(ns) * K;
    const uint64_t blocks = min_u64((total + 255) / 256, 148ull * 8);
    cell_sizes_kernel<<<static_cast<unsigned>(blocks ? blocks : 1), 256, 0, st>>>(cell_off, ns, K, cell_size);
    return cudaGetLastError();
}

cudaError_t launch_check_finite(const float* data, uint64_t count, int* flag, cudaStream_t st) {
    // `flag` points at an unsigned long long initialised to ~0 by the caller
    const uint64_t blocks = min_u64((count + 255) / 256, 148ull * 16);
    check_finite_kernel<<<static_cast<unsigned>(blocks ? blocks : 1), 256, 0, st>>>(
        data, count, reinterpret_cast<unsigned long long*>(flag));
    return cudaGetLastError();
}

namespace {
int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v && *v ? std::atoi(v) : dflt;
}
}  // namespace

Tuning tuning_from_env() {
    Tuning t;
    const int c = env_int("SUCO_CLUSTER", 0);
    t.cluster = (c >= 1 && c <= 16) ? c : 0;
    t.no_u8 = std::getenv("SUCO_NO_U8") != nullptr;
    const int q8 = env_int("SUCO_Q8", 1);
    t.q8 = q8 == 0 || q8 == 2 ? q8 : 1;
    const int qp = env_int("SUCO_Q8_PREFIX", 3);
    t.q8_prefix = (qp == 0 || qp == 1 || qp == 3) ? static_cast<uint32_t>(qp) : 3u;
    t.dense = env_int("SUCO_DENSE", 1) != 0;
    t.dense_half = env_int("SUCO_DENSE_HALF", 1);
    t.dense_pair = env_int("SUCO_DENSE_PAIR", 0);
    const int ds = env_int("SUCO_DENSE_SCHED", 1);
    t.dense_sched = ds >= 0 && ds <= 16 ? static_cast<uint32_t>(ds) : 1u;
    t.dense_fused = env_int("SUCO_DENSE_FUSED", 1) != 0;
    t.dense_stage = std::getenv("SUCO_DENSE_STAGE") != nullptr;
    const int b = env_int("SUCO_DENSE_BUF", 0);
    t.dense_buf = b > 0 ? static_cast<uint32_t>(b < 8 ? 8 : b / 8 * 8) : 0u;
    t.dense_nocut = std::getenv("SUCO_DENSE_NOCUT") != nullptr;
    if (const char* tc = std::getenv("SUCO_TIE_CUT")) {
        float sc = 0.f;
        unsigned pad = 0;
        if (std::sscanf(tc, "%f,%u", &sc, &pad) == 2 && sc >= 1.f && sc <= 4.f) {
            t.tie_cut_scale = sc;
            t.tie_cut_pad = pad;
        }
    }
    const int w = env_int("SUCO_DENSE_WORDS", 0);
    t.dense_words = (w == 1 || w == 2) ? static_cast<uint32_t>(w) : 0u;
    t.dense_stats = std::getenv("SUCO_DENSE_STATS") != nullptr;
    const int cm = env_int("SUCO_DENSE_COMPACT", 0);
    t.dense_compact = (cm == 1 || cm == 2) ? static_cast<uint32_t>(cm) : 0u;
    const int cr = env_int("SUCO_DENSE_COMPACT_ROWS", 0);
    t.dense_compact_rows = cr > 0 ? static_cast<uint32_t>(cr) : 0u;
    const int dp = env_int("SUCO_DENSE_PIECE", 0);
    t.dense_piece = dp >= 2048 && dp <= 32768 && dp % 2048 == 0 ? static_cast<uint32_t>(dp) : 0u;
    t.rerank_stats = std::getenv("SUCO_RERANK_STATS") != nullptr;
    const int tl = env_int("SUCO_TILES", 1);
    t.tiles = tl > 1 ? static_cast<uint32_t>(tl) : 1u;
    const char* mb = std::getenv("SUCO_SCRATCH_MB");
    t.scratch_bytes = mb && std::atoll(mb) > 0 ? static_cast<uint64_t>(std::atoll(mb)) << 20 : 0;
    t.fb_overlap = std::getenv("SUCO_FB_OVERLAP") ? (env_int("SUCO_FB_OVERLAP", 0) != 0) : -1;
    const char* tv = std::getenv("SUCO_TRAVERSE");
    t.traverse = tv && (tv[0] == 'w' || tv[0] == 's' || tv[0] == 'n' || tv[0] == 't' || tv[0] == 'r') ? tv[0] : 0;
    t.rerank_u8_regs = env_int("SUCO_RERANK_U8_PIPE", 1) == 0;
    t.rerank_tma = env_int("SUCO_RERANK_TMA", 0) != 0;
    const int rp = env_int("SUCO_RERANK_PIPE", 2);
    t.rerank_pipe = (rp == 0 || rp == 1) ? rp : 2;
    t.kpp_serial = env_int("SUCO_KPP_SERIAL", 0) == 1;
    const int scb = env_int("SUCO_SC_BATCH", 0);
    t.sc_batch = scb > 0 ? static_cast<uint32_t>(scb) : 0u;
    const char* ch = std::getenv("SUCO_BUILD_CHUNK");
    t.build_chunk = ch && std::atoll(ch) > 0 ? static_cast<uint64_t>(std::atoll(ch)) : 0;
    return t;
}

}  // namespace suco_gpu
