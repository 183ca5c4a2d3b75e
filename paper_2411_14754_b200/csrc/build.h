// Index build on the device (index.cpp:98-145, kmeans.cpp:58-194, index.cpp:69-96).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "index_format.h"
#include "tuning.h"

struct suco_comm;

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
                        const suco_index_params& p, BuildOutputs& out, cudaStream_t st, const Tuning& tune,
                        const uint32_t* train = nullptr, uint64_t n_train = 0);

// The sharded build (SURVEY §8(e) "Build"; index.cpp:118-137 over G ranks of `comm`): rank r
// holds the rows of global blocks j = r (mod G) (block size b) back to back, n_local of them.
// Job j's projected training column (all rows, or the ascending global ids train[0..n_train))
// is gathered in global id order on rank j % G, which runs that k-means; every job's centroids
// are broadcast; each rank assigns its own rows (kmeans.cpp:19-33) and builds its local IMI
// (local ids, ascending per cell: out.cell_off / out.ids over n_local); the per-cell counts are
// all-reduced into cell_size (device, ns x K): the global sizes.
void build_shard_device(const float* d_rows, uint64_t n_local, uint64_t n_global, uint32_t d, uint32_t b,
                        const HostLayout& L, const suco_index_params& p, suco_comm* comm, BuildOutputs& out,
                        uint32_t* cell_size, cudaStream_t st, const Tuning& tune, const uint32_t* train = nullptr,
                        uint64_t n_train = 0);

// Stand-alone kmeans / build_imi on host buffers (parity entry points).
void kmeans_device_host_io(const float* points, uint64_t n, uint32_t dim, uint32_t k, uint32_t iterations,
                           uint64_t seed, float* centroids, uint32_t* assignments, uint32_t* repaired,
                           uint32_t* num_repaired);
void build_imi_host_io(const uint32_t* first, const uint32_t* second, uint64_t n, uint32_t k_half,
                       uint64_t* offsets, uint32_t* ids);

}  // namespace suco_gpu
