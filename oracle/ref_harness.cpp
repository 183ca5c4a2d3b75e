// TEST INFRASTRUCTURE ONLY — never part of the product path.
//
// C-linkage harness over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp + tests/support/*.cpp), compiled by
// oracle/Makefile into oracle/_ref/libsuco_ref.so. It lets the Python tests
// and bench.py's CPU-baseline arm drive the reference's own public API:
//   build_index      index.hpp:85      (index.cpp:98-145)
//   knn_query        query.hpp:93-96   (query.cpp:199-262)
//   run_suco_batch   suco_cli.cpp:95-114 (timing definition of QPS)
//   centroid_distances / dynamic_activation / multi_sequence / rerank
//                    query.hpp:27-84
//   kmeans           kmeans.hpp:46-48
//   build_imi        index.hpp:38-39
//   serialize_index / deserialize_index   index.hpp:99-108
//   collision_count / candidate_count     sc_linear.hpp:36-40
//   testsupport::clustered / uniform / random_* / exhaustive_traversal
//                    tests/support/synthetic.hpp, oracles.hpp
// No reference source is copied here; everything below is glue.

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "suco/core.hpp"
#include "suco/eval.hpp"
#include "suco/index.hpp"
#include "suco/io.hpp"
#include "suco/kmeans.hpp"
#include "suco/parallel.hpp"
#include "suco/query.hpp"
#include "suco/rng.hpp"
#include "suco/sc_linear.hpp"
#include "suco/subspace.hpp"
#include "support/oracles.hpp"
#include "support/synthetic.hpp"

namespace {

thread_local std::string g_err;

// Status codes shared with include/suco_b200.h.
int code_of(const std::exception_ptr& ep) {
    try {
        std::rethrow_exception(ep);
    } catch (const suco::CorruptIndexError& e) {
        g_err = e.what();
        return 3;
    } catch (const suco::FormatError& e) {
        g_err = e.what();
        return 3;
    } catch (const suco::ConfigError& e) {
        g_err = e.what();
        return 2;
    } catch (const suco::IncompatibilityError& e) {
        g_err = e.what();
        return 4;
    } catch (const suco::ContractError& e) {
        g_err = e.what();
        return 5;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    } catch (...) {
        g_err = "unknown exception";
        return 1;
    }
}

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

suco::Dataset make_dataset(const float* data, std::uint64_t n, std::uint32_t d) {
    return suco::Dataset(n, d, std::vector<float>(data, data + n * static_cast<std::uint64_t>(d)));
}

suco::CentroidDistances make_cd(const double* dists, const std::uint32_t* order, std::uint32_t k) {
    suco::CentroidDistances cd;
    cd.dists.assign(dists, dists + k);
    cd.order.assign(order, order + k);
    return cd;
}

suco::Imi make_imi(std::uint32_t k_half, const std::uint64_t* offsets, const std::uint32_t* ids,
                   std::uint64_t n) {
    suco::Imi imi;
    imi.k_half = k_half;
    const std::uint64_t cells = static_cast<std::uint64_t>(k_half) * k_half;
    imi.offsets.assign(offsets, offsets + cells + 1);
    imi.ids.assign(ids, ids + n);
    return imi;
}

int write_cells(const suco::RetrievedClusters& r, std::uint32_t* c1, std::uint32_t* c2,
                std::uint64_t* cum, double* sums, std::uint64_t cap, std::uint64_t* count) {
    *count = r.cells.size();
    if (r.cells.size() > cap) {
        g_err = "cell output capacity too small";
        return 5;
    }
    for (std::size_t i = 0; i < r.cells.size(); ++i) {
        c1[i] = r.cells[i].c1;
        c2[i] = r.cells[i].c2;
        cum[i] = r.cells[i].cumulative;
        sums[i] = r.cells[i].sum_dist;
    }
    return 0;
}

struct RefIndex {
    suco::SucoIndex index;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- rng / KATs
std::uint64_t ref_splitmix64(std::uint64_t x) { return suco::splitmix64(x); }
std::uint64_t ref_derive_seed(std::uint64_t s, std::uint64_t t) { return suco::derive_seed(s, t); }
std::uint64_t ref_fnv1a(const void* p, std::uint64_t len, std::uint64_t seed) {
    return suco::fnv1a(p, len, seed);
}
std::uint64_t ref_collision_count(double alpha, std::uint64_t n) {
    return suco::collision_count(alpha, n);
}
std::uint64_t ref_candidate_count(double beta, std::uint64_t n, std::uint64_t k) {
    return suco::candidate_count(beta, n, k);
}
int ref_validate_params(double alpha, double beta, std::uint32_t k, std::uint64_t n) {
    return guarded([&] {
        suco::CollisionParams p;
        p.alpha = alpha;
        p.beta = beta;
        p.k = k;
        p.validate(n);
    });
}

// ------------------------------------------------------------ synthetic data
int ref_clustered(std::uint64_t n, std::uint32_t d, std::uint32_t clusters, std::uint64_t seed,
                  double lo, double hi, double sigma, int quantize, float* out) {
    return guarded([&] {
        const suco::Dataset ds =
            suco::testsupport::clustered(n, d, clusters, seed, lo, hi, sigma, quantize != 0);
        std::memcpy(out, ds.data(), n * d * sizeof(float));
    });
}

int ref_uniform(std::uint64_t n, std::uint32_t d, std::uint64_t seed, float lo, float hi,
                float* out) {
    return guarded([&] {
        const suco::Dataset ds = suco::testsupport::uniform(n, d, seed, lo, hi);
        std::memcpy(out, ds.data(), n * d * sizeof(float));
    });
}

// io.cpp:212-252. base_out holds (n-count) x d, query_out count x d.
int ref_hold_out(const float* data, std::uint64_t n, std::uint32_t d, std::uint64_t count,
                 std::uint64_t seed, float* base_out, float* query_out) {
    return guarded([&] {
        const suco::Dataset ds = make_dataset(data, n, d);
        suco::HoldOutSplit split = suco::hold_out_queries(ds, count, seed);
        std::memcpy(base_out, split.base.data(), split.base.size() * d * sizeof(float));
        if (split.queries) {
            std::memcpy(query_out, split.queries->data(), count * d * sizeof(float));
        }
    });
}

// ---------------------------------------------------------------- geometry
int ref_sample_subspaces(std::uint32_t d, std::uint32_t ns, std::uint32_t mode,
                         std::uint64_t seed, std::uint32_t* dims_out, std::uint32_t* sizes_out,
                         std::uint32_t* split_out) {
    return guarded([&] {
        const suco::SubspaceLayout l =
            suco::sample_subspaces(d, ns, static_cast<suco::SubspaceMode>(mode), seed);
        std::size_t p = 0;
        for (std::uint32_t i = 0; i < ns; ++i) {
            sizes_out[i] = static_cast<std::uint32_t>(l.subspaces[i].size());
            split_out[i] = l.half_split[i];
            for (const auto v : l.subspaces[i]) dims_out[p++] = v;
        }
    });
}

// ------------------------------------------------------------------- build
int ref_kmeans(const float* points, std::uint64_t n, std::uint32_t dim, std::uint32_t k,
               std::uint32_t iters, std::uint64_t seed, unsigned threads, float* centroids,
               std::uint32_t* assign, std::uint32_t* repaired, std::uint32_t* nrepaired,
               double* wcss /* iters, may be null */) {
    return guarded([&] {
        suco::KMeansStats st;
        const suco::KMeansModel m =
            suco::kmeans(points, n, dim, k, iters, seed, threads, wcss ? &st : nullptr);
        std::memcpy(centroids, m.centroids.data(), m.centroids.size() * sizeof(float));
        std::memcpy(assign, m.assignments.data(), n * sizeof(std::uint32_t));
        *nrepaired = static_cast<std::uint32_t>(m.repaired.size());
        for (std::size_t i = 0; i < m.repaired.size(); ++i) repaired[i] = m.repaired[i];
        if (wcss) {
            for (std::size_t i = 0; i < st.wcss.size(); ++i) wcss[i] = st.wcss[i];
        }
    });
}

int ref_build_imi(const std::uint32_t* first, const std::uint32_t* second, std::uint64_t n,
                  std::uint32_t k_half, std::uint64_t* offsets, std::uint32_t* ids) {
    return guarded([&] {
        const suco::Imi imi = suco::build_imi({first, n}, {second, n}, k_half);
        std::memcpy(offsets, imi.offsets.data(), imi.offsets.size() * sizeof(std::uint64_t));
        std::memcpy(ids, imi.ids.data(), n * sizeof(std::uint32_t));
    });
}

int ref_build_index(const float* data, std::uint64_t n, std::uint32_t d, std::uint32_t ns,
                    std::uint32_t k_half, std::uint32_t iters, std::uint64_t seed,
                    std::uint32_t mode, unsigned threads, void** out) {
    return guarded([&] {
        const suco::Dataset ds = make_dataset(data, n, d);
        suco::IndexParams p;
        p.num_subspaces = ns;
        p.k_half = k_half;
        p.iterations = iters;
        p.seed = seed;
        p.mode = static_cast<suco::SubspaceMode>(mode);
        auto idx = std::make_unique<RefIndex>();
        idx->index = suco::build_index(ds, p, threads);
        *out = idx.release();
    });
}

int ref_index_from_bytes(const unsigned char* bytes, std::uint64_t len, void** out) {
    return guarded([&] {
        auto idx = std::make_unique<RefIndex>();
        idx->index = suco::deserialize_index({bytes, len});
        *out = idx.release();
    });
}

void ref_index_free(void* h) { delete static_cast<RefIndex*>(h); }

// Two-call protocol: buf == nullptr returns the size only.
int ref_index_serialize(void* h, unsigned char* buf, std::uint64_t cap, std::uint64_t* len) {
    return guarded([&] {
        const auto bytes = suco::serialize_index(static_cast<RefIndex*>(h)->index);
        *len = bytes.size();
        if (buf) {
            if (cap < bytes.size()) throw suco::ContractError("serialize: buffer too small");
            std::memcpy(buf, bytes.data(), bytes.size());
        }
    });
}

// -------------------------------------------------------------------- query
int ref_centroid_distances(const float* half_query, std::uint32_t dim, const float* centroids,
                           std::uint32_t k_half, double* dists, std::uint32_t* order) {
    return guarded([&] {
        const auto cd = suco::centroid_distances(
            {half_query, dim}, {centroids, static_cast<std::size_t>(k_half) * dim}, k_half);
        std::copy(cd.dists.begin(), cd.dists.end(), dists);
        std::copy(cd.order.begin(), cd.order.end(), order);
    });
}

// kind: 0 dynamic_activation, 1 multi_sequence, 2 testsupport::exhaustive_traversal
int ref_traverse(int kind, double alpha, std::uint64_t n, const double* d1, const std::uint32_t* o1,
                 const double* d2, const std::uint32_t* o2, std::uint32_t k_half,
                 const std::uint64_t* offsets, const std::uint32_t* ids, std::uint32_t* c1,
                 std::uint32_t* c2, std::uint64_t* cum, double* sums, std::uint64_t cap,
                 std::uint64_t* count) {
    int rc = 0;
    const int g = guarded([&] {
        const auto cd1 = make_cd(d1, o1, k_half);
        const auto cd2 = make_cd(d2, o2, k_half);
        const std::uint64_t total = offsets[static_cast<std::uint64_t>(k_half) * k_half];
        const suco::Imi imi = make_imi(k_half, offsets, ids, total);
        suco::RetrievedClusters r;
        if (kind == 0) r = suco::dynamic_activation(alpha, n, cd1, cd2, imi);
        else if (kind == 1) r = suco::multi_sequence(alpha, n, cd1, cd2, imi);
        else r = suco::testsupport::exhaustive_traversal(alpha, n, cd1, cd2, imi);
        rc = write_cells(r, c1, c2, cum, sums, cap, count);
    });
    return g ? g : rc;
}

int ref_rerank(const float* data, std::uint64_t n, std::uint32_t d, const float* query,
               std::uint32_t qlen, const std::uint32_t* cands, std::uint64_t m, std::uint32_t k,
               std::uint32_t* ids, double* dists, std::uint32_t* count) {
    return guarded([&] {
        const suco::Dataset ds = make_dataset(data, n, d);
        const auto r = suco::rerank(ds, {query, qlen}, {cands, m}, k);
        *count = static_cast<std::uint32_t>(r.entries.size());
        for (std::size_t i = 0; i < r.entries.size(); ++i) {
            ids[i] = r.entries[i].id;
            dists[i] = r.entries[i].distance;
        }
    });
}

int ref_exact_knn(const float* data, std::uint64_t n, std::uint32_t d, const float* query,
                  std::uint32_t k, std::uint32_t* ids, double* dists) {
    return guarded([&] {
        const suco::Dataset ds = make_dataset(data, n, d);
        const auto r = suco::exact_knn(ds, {query, d}, k);
        for (std::size_t i = 0; i < r.entries.size(); ++i) {
            ids[i] = r.entries[i].id;
            dists[i] = r.entries[i].distance;
        }
    });
}

// A dataset handle so repeated queries don't re-copy n x d floats.
int ref_dataset_new(const float* data, std::uint64_t n, std::uint32_t d, void** out) {
    return guarded([&] { *out = new suco::Dataset(make_dataset(data, n, d)); });
}
void ref_dataset_free(void* h) { delete static_cast<suco::Dataset*>(h); }

// Batched knn_query exactly like run_suco_batch (suco_cli.cpp:95-114):
// parallel_chunks over queries, thread_local QueryScratch, steady_clock wall.
// ids/dists are nq x k; counts[q] = entries returned. Returns wall seconds
// through *wall_s.
int ref_knn_query_batch(void* hidx, void* hdata, const float* queries, std::uint64_t nq,
                        std::uint32_t qlen, double alpha, double beta, std::uint32_t k,
                        int traversal, unsigned threads, std::uint32_t* ids, double* dists,
                        std::uint32_t* counts, double* wall_s) {
    return guarded([&] {
        const auto& index = static_cast<RefIndex*>(hidx)->index;
        const auto& ds = *static_cast<suco::Dataset*>(hdata);
        suco::CollisionParams p;
        p.alpha = alpha;
        p.beta = beta;
        p.k = k;
        const auto kind = traversal == 0 ? suco::TraversalKind::DynamicActivation
                                         : suco::TraversalKind::MultiSequence;
        const auto t0 = std::chrono::steady_clock::now();
        suco::parallel_chunks(nq, threads, 1, [&](std::size_t, std::size_t lo, std::size_t hi) {
            thread_local suco::QueryScratch scratch;
            for (std::size_t qi = lo; qi < hi; ++qi) {
                const auto r = suco::knn_query(index, ds, {queries + qi * qlen, qlen}, p, kind,
                                               &scratch);
                counts[qi] = static_cast<std::uint32_t>(r.entries.size());
                for (std::size_t i = 0; i < r.entries.size(); ++i) {
                    ids[qi * k + i] = r.entries[i].id;
                    dists[qi * k + i] = r.entries[i].distance;
                }
            }
        });
        *wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

// Per-query intermediates of knn_query, rebuilt from the reference's public
// stage functions in the same order as query.cpp:220-253: u32 scores (n),
// the candidate set (m ids, ascending) and per-subspace retrieved-cell counts.
int ref_query_intermediates(void* hidx, void* hdata, const float* query, std::uint32_t qlen,
                            double alpha, double beta, std::uint32_t k, std::uint32_t* scores,
                            std::uint32_t* cands, std::uint64_t* m_out,
                            std::uint32_t* cells_per_subspace, std::uint64_t* cumulative) {
    return guarded([&] {
        const auto& index = static_cast<RefIndex*>(hidx)->index;
        const auto& ds = *static_cast<suco::Dataset*>(hdata);
        suco::check_compatible(index, ds);
        suco::CollisionParams p;
        p.alpha = alpha;
        p.beta = beta;
        p.k = k;
        p.validate(ds.size());
        const std::uint64_t n = ds.size();
        std::fill(scores, scores + n, 0u);
        std::vector<suco::PointId> touched;
        const auto& layout = index.layout;
        for (std::uint32_t si = 0; si < layout.num_subspaces; ++si) {
            const auto& cb = index.subspaces[si];
            const auto q1 = suco::project({query, qlen}, layout, si, suco::Half::First);
            const auto q2 = suco::project({query, qlen}, layout, si, suco::Half::Second);
            const auto cd1 = suco::centroid_distances(q1, cb.centroids_first, index.params.k_half);
            const auto cd2 = suco::centroid_distances(q2, cb.centroids_second, index.params.k_half);
            const auto r = suco::dynamic_activation(alpha, n, cd1, cd2, cb.imi);
            cells_per_subspace[si] = static_cast<std::uint32_t>(r.cells.size());
            cumulative[si] = r.cells.empty() ? 0 : r.cells.back().cumulative;
            for (const auto& c : r.cells) {
                for (const auto id : cb.imi.cell(c.c1, c.c2)) {
                    if (scores[id]++ == 0) touched.push_back(id);
                }
            }
        }
        const std::uint64_t m = suco::candidate_count(beta, n, k);
        std::vector<suco::PointId> c(touched);
        if (c.size() >= m) {
            const auto better = [&](suco::PointId a, suco::PointId b) {
                if (scores[a] != scores[b]) return scores[a] > scores[b];
                return a < b;
            };
            if (m < c.size()) {
                std::nth_element(c.begin(), c.begin() + static_cast<std::ptrdiff_t>(m), c.end(),
                                 better);
                c.resize(m);
            }
        } else {
            for (suco::PointId id = 0; c.size() < m && id < n; ++id) {
                if (scores[id] == 0) c.push_back(id);
            }
        }
        std::sort(c.begin(), c.end());
        *m_out = m;
        std::copy(c.begin(), c.end(), cands);
    });
}

// Index accessors for parity (SucoIndex fields, index.hpp:67-74).
int ref_index_info(void* h, std::uint64_t* n, std::uint32_t* d, std::uint32_t* ns,
                   std::uint32_t* k_half) {
    const auto& idx = static_cast<RefIndex*>(h)->index;
    *n = idx.n;
    *d = idx.layout.d;
    *ns = idx.params.num_subspaces;
    *k_half = idx.params.k_half;
    return 0;
}

int ref_index_subspace(void* h, std::uint32_t si, float* cent1, float* cent2,
                       std::uint64_t* offsets, std::uint32_t* ids) {
    return guarded([&] {
        const auto& cb = static_cast<RefIndex*>(h)->index.subspaces.at(si);
        if (cent1) std::copy(cb.centroids_first.begin(), cb.centroids_first.end(), cent1);
        if (cent2) std::copy(cb.centroids_second.begin(), cb.centroids_second.end(), cent2);
        if (offsets) std::copy(cb.imi.offsets.begin(), cb.imi.offsets.end(), offsets);
        if (ids) std::copy(cb.imi.ids.begin(), cb.imi.ids.end(), ids);
    });
}

// testsupport fakes (oracles.cpp:137-160) driven by a seeded mt19937_64 whose
// state is carried between calls by the caller-owned handle.
void* ref_rng_new(std::uint64_t seed) { return new std::mt19937_64(seed); }
void ref_rng_free(void* h) { delete static_cast<std::mt19937_64*>(h); }
std::uint64_t ref_rng_uniform_below(void* h, std::uint64_t bound) {
    return suco::uniform_below(*static_cast<std::mt19937_64*>(h), bound);
}
double ref_rng_uniform_unit(void* h) { return suco::uniform_unit(*static_cast<std::mt19937_64*>(h)); }

int ref_rng_centroid_distances(void* h, std::uint32_t k_half, int quantize, double* dists,
                               std::uint32_t* order) {
    return guarded([&] {
        const auto cd = suco::testsupport::random_centroid_distances(
            k_half, *static_cast<std::mt19937_64*>(h), quantize != 0);
        std::copy(cd.dists.begin(), cd.dists.end(), dists);
        std::copy(cd.order.begin(), cd.order.end(), order);
    });
}

int ref_rng_imi(void* h, std::uint32_t k_half, std::uint64_t n, std::uint64_t* offsets,
                std::uint32_t* ids) {
    return guarded([&] {
        const auto imi =
            suco::testsupport::random_imi(k_half, n, *static_cast<std::mt19937_64*>(h));
        std::copy(imi.offsets.begin(), imi.offsets.end(), offsets);
        std::copy(imi.ids.begin(), imi.ids.end(), ids);
    });
}

unsigned ref_hardware_threads() { return suco::effective_threads(0); }

// SC-Linear (sc_linear.hpp:45-53) over an index's layout and a dataset handle.
int ref_sc_scores(void* hidx, void* hdata, const float* query, std::uint32_t qlen, double alpha,
                  std::uint32_t* scores) {
    return guarded([&] {
        const auto& idx = static_cast<RefIndex*>(hidx)->index;
        const auto& ds = *static_cast<suco::Dataset*>(hdata);
        const auto sc = suco::compute_sc_scores(ds, idx.layout, {query, qlen}, alpha);
        for (std::size_t i = 0; i < sc.scores.size(); ++i) scores[i] = static_cast<std::uint32_t>(sc.scores[i]);
    });
}

int ref_sc_linear_query(void* hidx, void* hdata, const float* query, std::uint32_t qlen, double alpha,
                        double beta, std::uint32_t k, std::uint32_t* ids, double* dists, std::uint32_t* count) {
    return guarded([&] {
        const auto& idx = static_cast<RefIndex*>(hidx)->index;
        const auto& ds = *static_cast<suco::Dataset*>(hdata);
        const auto r = suco::sc_linear_query(ds, idx.layout, {query, qlen}, suco::CollisionParams{alpha, beta, k});
        for (std::size_t i = 0; i < r.entries.size(); ++i) {
            ids[i] = r.entries[i].id;
            dists[i] = r.entries[i].distance;
        }
        *count = static_cast<std::uint32_t>(r.entries.size());
    });
}

}  // extern "C"
