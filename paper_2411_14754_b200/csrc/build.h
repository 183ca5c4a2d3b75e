// Index build on the device (index.cpp:98-145, kmeans.cpp:58-194, index.cpp:69-96).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "index_format.h"

namespace suco_gpu {

struct BuildOutputs {
    uint32_t* cell_off;  // device, ns x (K+1) u32
    uint32_t* ids;       // device, ns x n
    std::vector<std::vector<float>>* cent1;  // host, ns
    std::vector<std::vector<float>>* cent2;
};

// All 2*N_s (subspace, half) k-means jobs run concurrently on one device,
// then one stable bucket sort per subspace emits the IMI CSR.
// train != nullptr (host, n_train strictly ascending row ids): the sampled build — k-means on
// those rows only, then every row assigned to its nearest centroid (kmeans.cpp:19-33).
void build_index_device(const float* d_data, uint64_t n, uint32_t d, const HostLayout& L,
                        const suco_index_params& p, BuildOutputs& out, cudaStream_t st,
                        const uint32_t* train = nullptr, uint64_t n_train = 0);

// Stand-alone kmeans / build_imi on host buffers (parity entry points).
void kmeans_device_host_io(const float* points, uint64_t n, uint32_t dim, uint32_t k, uint32_t iterations,
                           uint64_t seed, float* centroids, uint32_t* assignments, uint32_t* repaired,
                           uint32_t* num_repaired);
void build_imi_host_io(const uint32_t* first, const uint32_t* second, uint64_t n, uint32_t k_half,
                       uint64_t* offsets, uint32_t* ids);

}  // namespace suco_gpu
