// The communicator of the multi-GPU shard protocol.
//
// Two implementations behind one interface:
//   * NCCL (one process per GPU, NVLink 5 / NVSwitch): every collective is
//     enqueued on the caller's stream and returns at once;
//   * in-process (G shards driven by G host threads of one process, e.g. all
//     on one GPU for CI): each collective synchronises the caller's stream,
//     meets the other threads at a host barrier and copies the peers' device
//     buffers with cudaMemcpyAsync — no kernel ever waits on another rank.
// All buffers are device memory; `recv` of allgather / gather is rank-major
// (rank r's `bytes` at offset r * bytes).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

struct suco_comm {
    int rank = 0, size = 1;
    uint64_t bytes_sent = 0;  // running total of this rank's send volume (exchange accounting)
    virtual ~suco_comm() = default;
    virtual void allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) = 0;
    virtual void broadcast(void* buf, size_t bytes, int root, cudaStream_t st) = 0;
    virtual void allreduce_sum_u32(uint32_t* buf, size_t count, cudaStream_t st) = 0;
    virtual void gather(const void* send, void* recv, size_t bytes, int root, cudaStream_t st) = 0;
    virtual const char* kind() const = 0;
};

namespace suco_gpu {

// Host-side agreement on one status code across ranks (max over ranks; a failing rank's error
// reaches every rank instead of leaving the others blocked in the next collective).
int agree_status(suco_comm* comm, int code, cudaStream_t st);
// max over ranks of a host u64 (all ranks must take the same tile count, etc.)
uint64_t agree_max(suco_comm* comm, uint64_t v, cudaStream_t st);

}  // namespace suco_gpu
