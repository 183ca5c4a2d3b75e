// suco_b200.hpp — C++ mirror of the reference API (/root/reference/proj/include/suco)
// over the C-ABI of libsuco_b200.so. Same names, argument meaning, defaults and
// exception taxonomy as the reference, so code written against suco:: can move
// to suco::gpu:: by changing the namespace:
//
//   reference                                   here
//   suco::build_index      index.hpp:85         suco::gpu::build_index          -> suco_gpu_build_index
//   suco::load_index/deserialize index.hpp:101-107  suco::gpu::load_index         -> suco_gpu_load_index
//   suco::serialize_index  index.hpp:99         suco::gpu::serialize_index      -> suco_gpu_serialize_index
//   suco::knn_query        query.hpp:93-96      suco::gpu::knn_query(_batch)    -> suco_gpu_knn_query_batch(_device)
//   suco::centroid_distances query.hpp:27       suco::gpu::centroid_distances   -> suco_gpu_centroid_distances
//   suco::dynamic_activation query.hpp:57       suco::gpu::dynamic_activation   -> suco_gpu_dynamic_activation
//   suco::rerank           query.hpp:83         suco::gpu::rerank               -> suco_gpu_rerank
//   suco::kmeans           kmeans.hpp:46        suco::gpu::kmeans               -> suco_gpu_kmeans
//   suco::build_imi        index.hpp:39         suco::gpu::build_imi            -> suco_gpu_build_imi
//   suco::collision_count / candidate_count / CollisionParams::validate (sc_linear.hpp:30-40)
//                                               -> suco_collision_count / suco_candidate_count /
//                                                  suco_validate_collision_params
//   suco::QueryScratch     query.hpp:72-78      suco::gpu::QueryScratch         -> suco_gpu_query_ctx_create /
//                                                  suco_gpu_query_ctx_free / suco_gpu_query_ctx_synchronize /
//                                                  suco_gpu_query_ctx_set_profiling / suco_gpu_query_ctx_stage_times /
//                                                  suco_gpu_query_ctx_last_launches / suco_gpu_query_ctx_exchange_bytes
// Multi-GPU shard protocol (no reference counterpart; the sharded build_index / knn_query):
//   suco::gpu::Comm  -> suco_comm_nccl_id / suco_comm_nccl_create / suco_comm_local_create /
//                       suco_comm_info / suco_comm_free
//   suco::gpu::build_shard / make_shard / shard_block_hint / GpuIndex::shard_info /
//   GpuIndex::shard_knn_query_batch(_device)
//                    -> suco_gpu_build_shard / suco_gpu_make_shard / suco_gpu_shard_block_hint /
//                       suco_gpu_shard_info / suco_gpu_shard_knn_query_batch(_device)
// Also wrapped: suco_last_error, suco_gpu_device_count, suco_gpu_index_info,
// suco_gpu_index_subspace, suco_gpu_free_index, suco_gpu_query_intermediates,
// suco_gpu_exact_knn_batch (GpuIndex::exact_knn_batch; recall / mre as in eval.cpp:64-102),
// suco_gpu_sc_scores / suco_gpu_sc_linear_batch (GpuIndex::sc_scores / sc_linear_batch, sc_linear.hpp:45-53),
// suco_read_vecs / suco_write_vecs / suco_gpu_build_index_from_vecs / suco_gpu_load_index_from_vecs
// (vecs I/O, io.hpp:22-40; raw C entry points).
#pragma once

#include <cstdint>
#include <limits>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "suco_b200.h"

namespace suco::gpu {

// error.hpp:9-37
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ContractError : Error {
    using Error::Error;
};
struct ConfigError : Error {
    using Error::Error;
};
struct FormatError : Error {
    using Error::Error;
};
struct CorruptIndexError : FormatError {
    using FormatError::FormatError;
};
struct IncompatibilityError : Error {
    using Error::Error;
};

inline void check(int rc) {
    if (rc == SUCO_OK) return;
    const std::string msg = suco_last_error();
    switch (rc) {
        case SUCO_ERR_CONFIG: throw ConfigError(msg);
        case SUCO_ERR_FORMAT: throw FormatError(msg);
        case SUCO_ERR_CORRUPT_INDEX: throw CorruptIndexError(msg);
        case SUCO_ERR_INCOMPATIBLE: throw IncompatibilityError(msg);
        case SUCO_ERR_CONTRACT: throw ContractError(msg);
        default: throw Error(msg);
    }
}

using PointId = std::uint32_t;
enum class SubspaceMode : std::uint32_t { Contiguous = 0, Shuffled = 1 };

struct IndexParams {  // index.hpp:53-61
    std::uint32_t num_subspaces = 8;
    std::uint32_t k_half = 50;
    std::uint32_t iterations = 10;
    std::uint64_t seed = 42;
    SubspaceMode mode = SubspaceMode::Contiguous;
    suco_index_params c() const {
        return {num_subspaces, k_half, iterations, static_cast<std::uint32_t>(mode), seed};
    }
};

struct CollisionParams {  // sc_linear.hpp:22-31
    double alpha = 0.05;
    double beta = 0.005;
    std::uint32_t k = 50;
    suco_collision_params c() const { return {alpha, beta, k}; }
    void validate(std::uint64_t n) const {
        const auto p = c();
        check(suco_validate_collision_params(&p, n));
    }
};

inline std::uint64_t collision_count(double alpha, std::uint64_t n) { return suco_collision_count(alpha, n); }
inline std::uint64_t candidate_count(double beta, std::uint64_t n, std::uint64_t k) {
    return suco_candidate_count(beta, n, k);
}

struct Neighbor {  // core.hpp:40-45
    PointId id;
    double distance;
    friend bool operator==(const Neighbor&, const Neighbor&) = default;
};
struct QueryResult {  // core.hpp:49-51
    std::vector<Neighbor> entries;
};
struct CentroidDistances {  // query.hpp:19-22
    std::vector<double> dists;
    std::vector<std::uint32_t> order;
};
struct RetrievedCell {  // query.hpp:33-40
    std::uint32_t c1, c2;
    std::uint64_t cumulative;
    double sum_dist;
    friend bool operator==(const RetrievedCell&, const RetrievedCell&) = default;
};
struct KMeansModel {  // kmeans.hpp:16-30
    std::uint32_t k = 0, dim = 0;
    std::vector<float> centroids;
    std::vector<std::uint32_t> assignments;
    std::vector<std::uint32_t> repaired;
};
struct Imi {  // index.hpp:19-34 (CSR form)
    std::uint32_t k_half = 0;
    std::vector<std::uint64_t> offsets;
    std::vector<PointId> ids;
};

inline int device_count() {
    int n = 0;
    check(suco_gpu_device_count(&n));
    return n;
}

class GpuIndex;

// Caller-owned query state (query.hpp:72-78): scratch, streams, events, profiling. One thread at a
// time; bound to the index it was made for.
class QueryScratch {
public:
    explicit QueryScratch(const GpuIndex& index);
    suco_gpu_query_ctx* handle() const { return h_.get(); }
    void synchronize() { check(suco_gpu_query_ctx_synchronize(h_.get())); }
    void set_profiling(bool on) { check(suco_gpu_query_ctx_set_profiling(h_.get(), on ? 1 : 0)); }
    // per-stage device ms of the last call {traverse, select, rerank}; stats {retrieved ids, nq, m}
    void stage_times(double ms[3], std::uint64_t stats[3]) { check(suco_gpu_query_ctx_stage_times(h_.get(), ms, stats)); }
    std::uint64_t last_launches() const {
        std::uint64_t n = 0;
        check(suco_gpu_query_ctx_last_launches(h_.get(), &n));
        return n;
    }
    std::uint64_t exchange_bytes() const {
        std::uint64_t n = 0;
        check(suco_gpu_query_ctx_exchange_bytes(h_.get(), &n));
        return n;
    }

private:
    std::unique_ptr<suco_gpu_query_ctx, void (*)(suco_gpu_query_ctx*)> h_;
};

// A member of the shard protocol's communicator (NCCL, or in-process for G threads).
class Comm {
public:
    explicit Comm(suco_comm* h) : h_(h, &suco_comm_free) {}
    static std::vector<unsigned char> nccl_id() {
        std::vector<unsigned char> id(SUCO_NCCL_ID_BYTES);
        check(suco_comm_nccl_id(id.data()));
        return id;
    }
    static Comm nccl(std::span<const unsigned char> id, int nranks, int rank, int device) {
        if (id.size() != SUCO_NCCL_ID_BYTES) throw ContractError("NCCL id must be SUCO_NCCL_ID_BYTES bytes");
        suco_comm* h = nullptr;
        check(suco_comm_nccl_create(id.data(), nranks, rank, device, &h));
        return Comm(h);
    }
    static std::vector<Comm> local(int nranks) {
        std::vector<suco_comm*> hs(static_cast<std::size_t>(nranks > 0 ? nranks : 0));
        check(suco_comm_local_create(nranks, hs.data()));
        std::vector<Comm> out;
        for (suco_comm* h : hs) out.emplace_back(h);
        return out;
    }
    suco_comm* handle() const { return h_.get(); }
    int rank() const {
        int r = 0;
        check(suco_comm_info(h_.get(), &r, nullptr, nullptr));
        return r;
    }
    int size() const {
        int s = 0;
        check(suco_comm_info(h_.get(), nullptr, &s, nullptr));
        return s;
    }

private:
    std::unique_ptr<suco_comm, void (*)(suco_comm*)> h_;
};

inline std::uint32_t shard_block_hint(std::uint64_t n, std::uint32_t num_shards) {
    std::uint32_t b = 0;
    check(suco_gpu_shard_block_hint(n, num_shards, &b));
    return b;
}

inline std::uint32_t batch_qlen(std::span<const float> queries, std::uint64_t nq) {
    if (nq == 0) return 0;
    if (queries.size() % nq != 0) throw ContractError("query buffer length is not a multiple of nq");
    return static_cast<std::uint32_t>(queries.size() / nq);
}

inline std::vector<QueryResult> to_results(const std::vector<std::uint32_t>& ids, const std::vector<double>& dists,
                                           std::uint64_t nq, std::uint32_t k) {
    std::vector<QueryResult> out(nq);
    for (std::uint64_t q = 0; q < nq; ++q) {
        out[q].entries.resize(k);
        for (std::uint32_t i = 0; i < k; ++i) out[q].entries[i] = {ids[q * k + i], dists[q * k + i]};
    }
    return out;
}

// Device-resident SucoIndex (+ the dataset rows it re-ranks), or one shard of it.
class GpuIndex {
public:
    explicit GpuIndex(suco_gpu_index* h) : h_(h, &suco_gpu_free_index) {}
    suco_gpu_index* handle() const { return h_.get(); }

    std::uint64_t n() const {
        std::uint64_t n = 0;
        check(suco_gpu_index_info(h_.get(), &n, nullptr, nullptr, nullptr, nullptr, nullptr));
        return n;
    }
    std::uint32_t dim() const {
        std::uint32_t d = 0;
        check(suco_gpu_index_info(h_.get(), nullptr, &d, nullptr, nullptr, nullptr, nullptr));
        return d;
    }
    IndexParams params() const {
        suco_index_params p{};
        check(suco_gpu_index_info(h_.get(), nullptr, nullptr, &p, nullptr, nullptr, nullptr));
        return {p.num_subspaces, p.k_half, p.iterations, p.seed, static_cast<SubspaceMode>(p.mode)};
    }
    Imi imi(std::uint32_t subspace) const {
        Imi m;
        m.k_half = params().k_half;
        m.offsets.resize(std::uint64_t(m.k_half) * m.k_half + 1);
        m.ids.resize(n());
        check(suco_gpu_index_subspace(h_.get(), subspace, nullptr, nullptr, m.offsets.data(), m.ids.data()));
        return m;
    }

    // run_suco_batch semantics (suco_cli.cpp:95-114): one QueryResult per row; queries.size() must
    // be nq x d. `scratch`: the caller's QueryScratch (query.hpp:96), or nullptr (pooled).
    std::vector<QueryResult> knn_query_batch(std::span<const float> queries, std::uint64_t nq,
                                             const CollisionParams& params, QueryScratch* scratch = nullptr) const {
        const auto cp = params.c();
        const std::uint32_t qlen = batch_qlen(queries, nq);
        std::vector<std::uint32_t> ids(nq * params.k);
        std::vector<double> dists(nq * params.k);
        check(suco_gpu_knn_query_batch(h_.get(), queries.data(), nq, qlen, &cp, ids.data(), dists.data(),
                                       scratch ? scratch->handle() : nullptr));
        return to_results(ids, dists, nq, params.k);
    }

    // The sharded knn_query: every rank of `comm` passes the same queries and gets the full result.
    std::vector<QueryResult> shard_knn_query_batch(const Comm& comm, std::span<const float> queries, std::uint64_t nq,
                                                   const CollisionParams& params,
                                                   QueryScratch* scratch = nullptr) const {
        const auto cp = params.c();
        const std::uint32_t qlen = batch_qlen(queries, nq);
        std::vector<std::uint32_t> ids(nq * params.k);
        std::vector<double> dists(nq * params.k);
        check(suco_gpu_shard_knn_query_batch(h_.get(), comm.handle(), queries.data(), nq, qlen, &cp, ids.data(),
                                             dists.data(), scratch ? scratch->handle() : nullptr));
        return to_results(ids, dists, nq, params.k);
    }
    void shard_knn_query_batch_device(const Comm& comm, const float* d_queries, std::uint64_t nq, std::uint32_t qlen,
                                      const CollisionParams& params, std::uint32_t* d_ids, double* d_dists,
                                      void* stream = nullptr, QueryScratch* scratch = nullptr) const {
        const auto cp = params.c();
        check(suco_gpu_shard_knn_query_batch_device(h_.get(), comm.handle(), d_queries, nq, qlen, &cp, d_ids, d_dists,
                                                    stream, scratch ? scratch->handle() : nullptr));
    }
    struct ShardInfo {
        std::uint64_t n_global = 0, n_local = 0;
        std::uint32_t block = 0, shard = 0, num_shards = 1;
    };
    ShardInfo shard_info() const {
        ShardInfo i;
        check(suco_gpu_shard_info(h_.get(), &i.n_global, &i.n_local, &i.block, &i.shard, &i.num_shards));
        return i;
    }

    // exact_knn (eval.hpp:29) for every row: the GPU ground truth, ascending by (distance, id).
    std::vector<QueryResult> exact_knn_batch(std::span<const float> queries, std::uint64_t nq, std::uint32_t k) const {
        const std::uint32_t qlen = batch_qlen(queries, nq);
        std::vector<std::uint32_t> ids(nq * k);
        std::vector<double> dists(nq * k);
        check(suco_gpu_exact_knn_batch(h_.get(), queries.data(), nq, qlen, k, ids.data(), dists.data()));
        return to_results(ids, dists, nq, k);
    }

    // compute_sc_scores (sc_linear.hpp:45-50) for one query: n per-point collision counts.
    std::vector<std::uint32_t> sc_scores(std::span<const float> query, double alpha) const {
        std::vector<std::uint32_t> scores(n());
        check(suco_gpu_sc_scores(h_.get(), query.data(), static_cast<std::uint32_t>(query.size()), alpha,
                                 scores.data()));
        return scores;
    }

    // sc_linear_query (sc_linear.hpp:52-53) for every row: the SC-Linear baseline.
    std::vector<QueryResult> sc_linear_batch(std::span<const float> queries, std::uint64_t nq,
                                             const CollisionParams& params) const {
        const std::uint32_t qlen = batch_qlen(queries, nq);
        std::vector<std::uint32_t> ids(nq * params.k);
        std::vector<double> dists(nq * params.k);
        const auto cp = params.c();
        check(suco_gpu_sc_linear_batch(h_.get(), queries.data(), nq, qlen, &cp, ids.data(), dists.data()));
        return to_results(ids, dists, nq, params.k);
    }

    // Device-resident queries/outputs (nq x qlen f32 in, nq x k u32/f64 out), enqueued on `stream`.
    void knn_query_batch_device(const float* d_queries, std::uint64_t nq, std::uint32_t qlen,
                                const CollisionParams& params, std::uint32_t* d_ids, double* d_dists,
                                void* stream = nullptr, QueryScratch* scratch = nullptr) const {
        const auto cp = params.c();
        check(suco_gpu_knn_query_batch_device(h_.get(), d_queries, nq, qlen, &cp, d_ids, d_dists, stream,
                                              scratch ? scratch->handle() : nullptr));
    }

    struct Intermediates {
        std::vector<std::uint32_t> scores, candidates, cells_per_subspace;
        std::vector<std::uint64_t> cumulative;
    };
    Intermediates query_intermediates(std::span<const float> query, const CollisionParams& params) const {
        const auto cp = params.c();
        Intermediates r;
        const auto p = this->params();
        r.scores.resize(n());
        r.candidates.resize(n());
        r.cells_per_subspace.resize(p.num_subspaces);
        r.cumulative.resize(p.num_subspaces);
        std::uint64_t m = 0;
        check(suco_gpu_query_intermediates(h_.get(), query.data(), static_cast<std::uint32_t>(query.size()), &cp,
                                           r.scores.data(), r.candidates.data(), &m, r.cells_per_subspace.data(),
                                           r.cumulative.data()));
        r.candidates.resize(m);
        return r;
    }

private:
    std::unique_ptr<suco_gpu_index, void (*)(suco_gpu_index*)> h_;
};

inline QueryScratch::QueryScratch(const GpuIndex& index) : h_(nullptr, &suco_gpu_query_ctx_free) {
    suco_gpu_query_ctx* c = nullptr;
    check(suco_gpu_query_ctx_create(index.handle(), &c));
    h_.reset(c);
}

// The sharded build_index: `rows` = this rank's rows (global blocks j = rank mod G, in order).
inline GpuIndex build_shard(std::span<const float> rows, std::uint64_t n_global, std::uint32_t d,
                            const IndexParams& params, std::uint32_t block, const Comm& comm, int device = 0,
                            std::span<const std::uint32_t> train_ids = {}) {
    const auto p = params.c();
    suco_gpu_index* h = nullptr;
    check(suco_gpu_build_shard(rows.data(), n_global, d, &p, block, train_ids.empty() ? nullptr : train_ids.data(),
                               train_ids.size(), comm.handle(), device, &h));
    return GpuIndex(h);
}

inline GpuIndex make_shard(const GpuIndex& full, std::uint32_t shard, std::uint32_t num_shards, std::uint32_t block) {
    suco_gpu_index* h = nullptr;
    check(suco_gpu_make_shard(full.handle(), shard, num_shards, block, &h));
    return GpuIndex(h);
}

inline GpuIndex build_index(std::span<const float> data, std::uint64_t n, std::uint32_t d,
                            const IndexParams& params = {}, int device = 0) {
    const auto p = params.c();
    suco_gpu_index* h = nullptr;
    check(suco_gpu_build_index(data.data(), n, d, &p, device, &h));
    return GpuIndex(h);
}

// Config 5's sampled build (suco_gpu_build_index_sampled).
inline GpuIndex build_index_sampled(std::span<const float> data, std::uint64_t n, std::uint32_t d,
                                    std::span<const std::uint32_t> train_ids, const IndexParams& params = {},
                                    int device = 0) {
    const auto p = params.c();
    suco_gpu_index* h = nullptr;
    check(suco_gpu_build_index_sampled(data.data(), n, d, &p, train_ids.data(), train_ids.size(), device, &h));
    return GpuIndex(h);
}

inline GpuIndex load_index(std::span<const unsigned char> bytes, std::span<const float> data, std::uint64_t n,
                           std::uint32_t d, int device = 0) {
    suco_gpu_index* h = nullptr;
    check(suco_gpu_load_index(bytes.data(), bytes.size(), data.data(), n, d, device, &h));
    return GpuIndex(h);
}

inline std::vector<unsigned char> serialize_index(const GpuIndex& index) {
    std::uint64_t len = 0;
    check(suco_gpu_serialize_index(index.handle(), nullptr, 0, &len));
    std::vector<unsigned char> b(len);
    check(suco_gpu_serialize_index(index.handle(), b.data(), b.size(), &len));
    return b;
}

// recall / mre (eval.hpp:33-39, eval.cpp:64-102): host arithmetic on one query's lists.
inline double recall(const QueryResult& result, std::span<const Neighbor> truth, std::uint32_t k) {
    if (k < 1) throw ContractError("recall: k must be >= 1");
    if (truth.size() < k) throw ContractError("recall: ground truth has fewer than k entries");
    if (result.entries.size() > k) throw ContractError("recall: result holds more than k entries");
    std::uint32_t hits = 0;
    for (const Neighbor& nb : result.entries) {
        for (std::uint32_t r = 0; r < k; ++r) hits += truth[r].id == nb.id;
    }
    return static_cast<double>(hits) / static_cast<double>(k);
}

inline double mre(const QueryResult& result, std::span<const Neighbor> truth, std::uint32_t k) {
    if (k < 1) throw ContractError("mre: k must be >= 1");
    if (truth.size() < k || result.entries.size() < k) throw ContractError("mre: both lists must hold at least k entries");
    double sum = 0.0;
    std::uint32_t included = 0;
    bool clean = true;
    for (std::uint32_t r = 0; r < k; ++r) {
        if (truth[r].distance == 0.0) {
            clean = clean && result.entries[r].distance == 0.0;
            continue;
        }
        sum += (result.entries[r].distance - truth[r].distance) / truth[r].distance;
        ++included;
    }
    if (included) return sum / included;
    return clean ? 0.0 : std::numeric_limits<double>::infinity();
}

inline QueryResult knn_query(const GpuIndex& index, std::span<const float> query, const CollisionParams& params) {
    return index.knn_query_batch(query, 1, params).front();
}

inline CentroidDistances centroid_distances(std::span<const float> half_query, std::span<const float> centroids,
                                            std::uint32_t k_half) {
    if (k_half >= 1 && !half_query.empty() && centroids.size() != std::size_t(k_half) * half_query.size()) {
        throw ContractError("centroid matrix does not match k_half x half dim");
    }
    CentroidDistances cd;
    cd.dists.resize(k_half);
    cd.order.resize(k_half);
    check(suco_gpu_centroid_distances(half_query.data(), static_cast<std::uint32_t>(half_query.size()),
                                      centroids.data(), k_half, cd.dists.data(), cd.order.data()));
    return cd;
}

inline std::vector<RetrievedCell> dynamic_activation(double alpha, std::uint64_t n, const CentroidDistances& cd1,
                                                     const CentroidDistances& cd2, const Imi& imi) {
    const std::uint64_t cap = std::uint64_t(imi.k_half) * imi.k_half;
    std::vector<std::uint32_t> c1(cap), c2(cap);
    std::vector<std::uint64_t> cum(cap);
    std::vector<double> sums(cap);
    std::uint64_t count = 0;
    check(suco_gpu_dynamic_activation(alpha, n, cd1.dists.data(), cd1.order.data(), cd2.dists.data(),
                                      cd2.order.data(), imi.k_half, imi.offsets.data(), c1.data(), c2.data(),
                                      cum.data(), sums.data(), cap, &count));
    std::vector<RetrievedCell> out(count);
    for (std::uint64_t i = 0; i < count; ++i) out[i] = {c1[i], c2[i], cum[i], sums[i]};
    return out;
}

inline QueryResult rerank(std::span<const float> data, std::uint64_t n, std::uint32_t d, std::span<const float> query,
                          std::span<const PointId> candidates, std::uint32_t k) {
    std::vector<std::uint32_t> ids(k);
    std::vector<double> dists(k);
    check(suco_gpu_rerank(data.data(), n, d, query.data(), static_cast<std::uint32_t>(query.size()),
                          candidates.data(), candidates.size(), k, ids.data(), dists.data()));
    QueryResult r;
    for (std::uint32_t i = 0; i < k; ++i) r.entries.push_back({ids[i], dists[i]});
    return r;
}

inline KMeansModel kmeans(const float* points, std::uint64_t n, std::uint32_t dim, std::uint32_t k,
                          std::uint32_t iterations, std::uint64_t seed, int device = 0) {
    KMeansModel m;
    m.k = k;
    m.dim = dim;
    m.centroids.resize(std::size_t(k) * dim);
    m.assignments.resize(n);
    m.repaired.resize(std::size_t(k) * iterations);
    std::uint32_t nrep = 0;
    check(suco_gpu_kmeans(points, n, dim, k, iterations, seed, device, m.centroids.data(), m.assignments.data(),
                          m.repaired.data(), &nrep));
    m.repaired.resize(nrep);
    return m;
}

inline Imi build_imi(std::span<const std::uint32_t> first, std::span<const std::uint32_t> second,
                     std::uint32_t k_half) {
    if (first.size() != second.size()) throw ContractError("assignment arrays differ in length");
    Imi imi;
    imi.k_half = k_half;
    imi.offsets.resize(std::uint64_t(k_half) * k_half + 1);
    imi.ids.resize(first.size());
    check(suco_gpu_build_imi(first.data(), second.data(), first.size(), k_half, imi.offsets.data(), imi.ids.data()));
    return imi;
}

}  // namespace suco::gpu
