// Ceiling of random record gathers on this GPU: N records of REC bytes, G gathers of the first
// BYTES bytes of uniformly random records (the re-rank's access pattern: 64-byte prefixes of int8
// records, 128-byte u8 rows), every load independent, 8 in flight per thread.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather_peak gather_peak.cu && ./gather_peak
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
    return static_cast<uint32_t>(x);
}

template <int GRAN>  // 16-byte granules read per record
__global__ void gather(const uint4* __restrict__ recs, uint32_t n, uint32_t rec_gran, uint64_t gathers, uint32_t* sink) {
    const uint64_t tid = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x, nthr = gridDim.x * uint64_t(blockDim.x);
    uint32_t acc = 0;
    // GRAN consecutive threads share a record
    for (uint64_t i = tid; i < gathers * GRAN; i += nthr * 8) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint64_t j = i + u * nthr;
            const uint32_t r = static_cast<uint32_t>((uint64_t(mix(j / GRAN)) * n) >> 32);
            v[u] = j < gathers * GRAN ? __ldcs(recs + uint64_t(r) * rec_gran + j % GRAN) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    if (acc == 0x12345678u) *sink = acc;
}

template <int GRAN>
static void run(const uint4* recs, uint32_t n, uint32_t rec_bytes, uint64_t gathers, uint32_t* sink) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e30f;
    for (int it = 0; it < 5; ++it) {
        cudaEventRecord(a);
        gather<GRAN><<<148 * 16, 256>>>(recs, n, rec_bytes / 16, gathers, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (it && ms < best) best = ms;
    }
    printf("{\"records\": %u, \"record_bytes\": %u, \"read_bytes\": %d, \"gathers\": %llu, \"ms\": %.3f, \"GBps\": %.1f}\n", n, rec_bytes,
           GRAN * 16, (unsigned long long)gathers, best, double(gathers) * GRAN * 16 / best / 1e6);
}

int main() {
    const uint32_t n = 10000000;
    uint32_t* sink; cudaMalloc(&sink, 4);
    for (uint32_t rec : {128u, 64u}) {
        uint4* recs; cudaMalloc(&recs, size_t(n) * rec); cudaMemset(recs, 1, size_t(n) * rec);
        const uint64_t g = 500000000ull;
        if (rec == 128) { run<4>(recs, n, rec, g, sink); run<8>(recs, n, rec, g, sink); run<2>(recs, n, rec, g, sink); }
        else { run<4>(recs, n, rec, g, sink); run<2>(recs, n, rec, g, sink); }
        cudaFree(recs);
    }
    return cudaGetLastError() != cudaSuccess;
}
