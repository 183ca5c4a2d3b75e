// Communicators of the shard protocol (comm.h): NCCL, and the in-process one.
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>

#include "capi_internal.h"
#include "comm.h"

using namespace suco_gpu;

namespace {

#define NCCL_TRY(x)                                                                                  \
    do {                                                                                             \
        const ncclResult_t r_ = (x);                                                                 \
        if (r_ != ncclSuccess) raise(SUCO_ERR_INTERNAL, std::string("NCCL error '") +              \
                                                            ncclGetErrorString(r_) + "' in " #x);    \
    } while (0)

struct NcclComm final : suco_comm {
    ncclComm_t c = nullptr;
    int device = 0;
    ~NcclComm() override {
        if (c) ncclCommDestroy(c);
    }
    void allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
        NCCL_TRY(ncclAllGather(send, recv, bytes, ncclUint8, c, st));
        bytes_sent += bytes;
    }
    void broadcast(void* buf, size_t bytes, int root, cudaStream_t st) override {
        NCCL_TRY(ncclBroadcast(buf, buf, bytes, ncclUint8, root, c, st));
        if (rank == root) bytes_sent += bytes;
    }
    void allreduce_sum_u32(uint32_t* buf, size_t count, cudaStream_t st) override {
        NCCL_TRY(ncclAllReduce(buf, buf, count, ncclUint32, ncclSum, c, st));
        bytes_sent += count * 4;
    }
    void gather(const void* send, void* recv, size_t bytes, int root, cudaStream_t st) override {
        NCCL_TRY(ncclGroupStart());
        if (rank == root) {
            for (int r = 0; r < size; ++r) {
                NCCL_TRY(ncclRecv(static_cast<char*>(recv) + size_t(r) * bytes, bytes, ncclUint8, r, c, st));
            }
        }
        NCCL_TRY(ncclSend(send, bytes, ncclUint8, root, c, st));
        NCCL_TRY(ncclGroupEnd());
        bytes_sent += bytes;
    }
    const char* kind() const override { return "nccl"; }
};

// Shared state of one in-process communicator (G member handles).
struct LocalShared {
    int G = 1;
    std::mutex mu;
    std::condition_variable cv;
    uint64_t gen = 0;
    int arrived = 0;
    bool poisoned = false;
    std::vector<const void*> ptr;
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        if (poisoned) raise(SUCO_ERR_INTERNAL, "another rank of the in-process communicator failed");
        const uint64_t g = gen;
        if (++arrived == G) {
            arrived = 0;
            ++gen;
            cv.notify_all();
            return;
        }
        cv.wait(lk, [&] { return gen != g || poisoned; });
        if (gen == g) raise(SUCO_ERR_INTERNAL, "another rank of the in-process communicator failed");
    }
    void poison() {
        std::lock_guard<std::mutex> lk(mu);
        poisoned = true;
        cv.notify_all();
    }
};

struct LocalComm final : suco_comm {
    std::shared_ptr<LocalShared> sh;
    // every collective: the caller's stream is drained, the buffers are posted, peers copy
    template <typename Fn>
    void exchange(const void* mine, cudaStream_t st, Fn&& copy) {
        try {
            CUDA_TRY(cudaStreamSynchronize(st));
            sh->ptr[rank] = mine;
            sh->barrier();
            copy();
            CUDA_TRY(cudaStreamSynchronize(st));
            sh->barrier();  // nobody rewrites a posted buffer before every peer has read it
        } catch (...) {
            sh->poison();
            throw;
        }
    }
    void allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
        exchange(send, st, [&] {
            for (int r = 0; r < size; ++r) {
                CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(recv) + size_t(r) * bytes, sh->ptr[r], bytes,
                                         cudaMemcpyDefault, st));
            }
        });
        bytes_sent += bytes;
    }
    void broadcast(void* buf, size_t bytes, int root, cudaStream_t st) override {
        exchange(buf, st, [&] {
            if (rank != root) CUDA_TRY(cudaMemcpyAsync(buf, sh->ptr[root], bytes, cudaMemcpyDefault, st));
        });
        if (rank == root) bytes_sent += bytes;
    }
    void allreduce_sum_u32(uint32_t* buf, size_t count, cudaStream_t st) override {
        DevBuf<uint32_t> all;
        all.reserve(count * size_t(size));
        allgather(buf, all.p, count * 4, st);
        CUDA_TRY(launch_sum_rows_u32(all.p, static_cast<uint32_t>(size), count, buf, st));
        CUDA_TRY(cudaStreamSynchronize(st));
    }
    void gather(const void* send, void* recv, size_t bytes, int root, cudaStream_t st) override {
        exchange(send, st, [&] {
            if (rank == root) {
                for (int r = 0; r < size; ++r) {
                    CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(recv) + size_t(r) * bytes, sh->ptr[r], bytes,
                                             cudaMemcpyDefault, st));
                }
            }
        });
        bytes_sent += bytes;
    }
    const char* kind() const override { return "local"; }
};

}  // namespace

namespace suco_gpu {

int agree_status(suco_comm* comm, int code, cudaStream_t st) {
    const uint64_t v = agree_max(comm, static_cast<uint64_t>(code < 0 ? 0 : code), st);
    return static_cast<int>(v);
}

uint64_t agree_max(suco_comm* comm, uint64_t v, cudaStream_t st) {
    if (comm->size == 1) return v;
    DevBuf<uint64_t> one, all;
    one.reserve(1);
    all.reserve(size_t(comm->size));
    CUDA_TRY(cudaMemcpyAsync(one.p, &v, 8, cudaMemcpyHostToDevice, st));
    comm->allgather(one.p, all.p, 8, st);
    std::vector<uint64_t> h(size_t(comm->size));
    CUDA_TRY(cudaMemcpyAsync(h.data(), all.p, h.size() * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    uint64_t mx = 0;
    for (uint64_t x : h) mx = std::max(mx, x);
    return mx;
}

}  // namespace suco_gpu

extern "C" {

int suco_comm_nccl_id(unsigned char* id) {
    return guarded([&] {
        if (!id) raise(SUCO_ERR_CONTRACT, "id buffer is null");
        ncclUniqueId u;
        NCCL_TRY(ncclGetUniqueId(&u));
        static_assert(sizeof(u.internal) == SUCO_NCCL_ID_BYTES, "NCCL unique id size");
        std::memcpy(id, u.internal, SUCO_NCCL_ID_BYTES);
    });
}

int suco_comm_nccl_create(const unsigned char* id, int nranks, int rank, int device, suco_comm** out) {
    return guarded([&] {
        if (!id || !out) raise(SUCO_ERR_CONTRACT, "null argument");
        *out = nullptr;
        if (nranks < 1 || rank < 0 || rank >= nranks) raise(SUCO_ERR_CONFIG, "rank must be in [0, nranks)");
        DeviceGuard g(device);
        ncclUniqueId u;
        std::memcpy(u.internal, id, SUCO_NCCL_ID_BYTES);
        auto c = std::make_unique<NcclComm>();
        c->rank = rank;
        c->size = nranks;
        c->device = device;
        NCCL_TRY(ncclCommInitRank(&c->c, nranks, u, rank));
        *out = c.release();
    });
}

int suco_comm_local_create(int nranks, suco_comm** out) {
    return guarded([&] {
        if (!out) raise(SUCO_ERR_CONTRACT, "null argument");
        if (nranks < 1 || nranks > 32) raise(SUCO_ERR_CONFIG, "in-process communicator: nranks must be in [1, 32]");
        auto sh = std::make_shared<LocalShared>();
        sh->G = nranks;
        sh->ptr.assign(size_t(nranks), nullptr);
        for (int r = 0; r < nranks; ++r) {
            auto c = new LocalComm();
            c->rank = r;
            c->size = nranks;
            c->sh = sh;
            out[r] = c;
        }
    });
}

int suco_comm_info(const suco_comm* comm, int* rank, int* size, uint64_t* bytes_sent) {
    return guarded([&] {
        if (!comm) raise(SUCO_ERR_CONTRACT, "communicator is null");
        if (rank) *rank = comm->rank;
        if (size) *size = comm->size;
        if (bytes_sent) *bytes_sent = comm->bytes_sent;
    });
}

void suco_comm_free(suco_comm* comm) { delete comm; }

}  // extern "C"
