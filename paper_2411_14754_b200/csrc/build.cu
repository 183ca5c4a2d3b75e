// Index build on the device — placeholder until the k-means kernels land.
#include "build.h"

namespace suco_gpu {

void build_index_device(const float*, uint64_t, uint32_t, const HostLayout&, const suco_index_params&, BuildOutputs&,
                        cudaStream_t) {
    raise(SUCO_ERR_INTERNAL, "GPU index build not implemented yet");
}

void kmeans_device_host_io(const float*, uint64_t, uint32_t, uint32_t, uint32_t, uint64_t, float*, uint32_t*, uint32_t*,
                           uint32_t*) {
    raise(SUCO_ERR_INTERNAL, "GPU kmeans not implemented yet");
}

void build_imi_host_io(const uint32_t*, const uint32_t*, uint64_t, uint32_t, uint64_t*, uint32_t*) {
    raise(SUCO_ERR_INTERNAL, "GPU build_imi not implemented yet");
}

}  // namespace suco_gpu
