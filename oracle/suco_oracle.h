/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the SuCo hot path.
 *
 * A plain-C restatement of the reference algorithm (/root/reference/proj),
 * written from its documented behaviour; every function cites the reference
 * file:line it restates. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it, and only as the checker. It is pinned against
 * the reference itself (oracle/_ref/libsuco_ref.so, compiled from the
 * reference sources) and the reference's known-answer tests in
 * tests/test_oracle.py.
 *
 * Status codes: 0 ok, 1 internal, 2 Config, 3 Format/CorruptIndex,
 * 4 Incompatibility, 5 Contract (mirrors include/suco_b200.h).
 */
#ifndef SUCO_ORACLE_H
#define SUCO_ORACLE_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct so_mt {
    uint64_t mt[312];
    int idx;
} so_mt;

const char* so_last_error(void);

/* rng.hpp:14-47 */
uint64_t so_splitmix64(uint64_t x);
uint64_t so_derive_seed(uint64_t seed, uint64_t stream);
void so_mt_seed(so_mt* g, uint64_t seed);
uint64_t so_mt_next(so_mt* g);
uint64_t so_uniform_below(so_mt* g, uint64_t bound);
double so_uniform_unit(so_mt* g);
double so_normal_unit(so_mt* g);
uint64_t so_fnv1a(const void* bytes, uint64_t len, uint64_t seed);

/* tests/support/synthetic.cpp:12-42, io.cpp:212-252 */
int so_clustered(uint64_t n, uint32_t d, uint32_t clusters, uint64_t seed, double lo, double hi,
                 double sigma, int quantize_u8, float* out);
int so_uniform(uint64_t n, uint32_t d, uint64_t seed, float lo, float hi, float* out);
int so_hold_out(const float* data, uint64_t n, uint32_t d, uint64_t count, uint64_t seed,
                float* base_out, float* query_out);

/* sc_linear.cpp:18-47 */
uint64_t so_collision_count(double alpha, uint64_t n);
uint64_t so_candidate_count(double beta, uint64_t n, uint64_t k);
int so_validate_params(double alpha, double beta, uint32_t k, uint64_t n);

/* subspace.cpp:10-44 */
int so_sample_subspaces(uint32_t d, uint32_t ns, uint32_t mode, uint64_t seed, uint32_t* dims_out,
                        uint32_t* sizes_out, uint32_t* split_out);

/* core.hpp:66-84 */
double so_sqdist4(const float* a, const float* b, size_t len);

/* kmeans.cpp:118-194 */
int so_kmeans(const float* points, uint64_t n, uint32_t dim, uint32_t k, uint32_t iters,
              uint64_t seed, float* centroids, uint32_t* assign, uint32_t* repaired,
              uint32_t* nrepaired, double* wcss);

/* index.cpp:69-96 */
int so_build_imi(const uint32_t* first, const uint32_t* second, uint64_t n, uint32_t k_half,
                 uint64_t* offsets, uint32_t* ids);

typedef struct so_index so_index;

/* index.cpp:98-145 ; `threads` jobs run concurrently, output independent of it */
int so_build_index(const float* data, uint64_t n, uint32_t d, uint32_t ns, uint32_t k_half,
                   uint32_t iters, uint64_t seed, uint32_t mode, unsigned threads, so_index** out);
/* Config 5's sampled build (BASELINE.json configs[4]; no reference API — composed from the
 * reference's own steps): the 2*N_s k-means jobs of index.cpp:120-137 run on the training rows
 * train[0..n_train) only (strictly ascending ids, in that order), then EVERY row is assigned to
 * its nearest centroid by kmeans.cpp:19-33's rule and build_imi (index.cpp:69-96) runs over all n.
 * With train = 0..n-1 it equals so_build_index. */
int so_build_index_sampled(const float* data, uint64_t n, uint32_t d, uint32_t ns, uint32_t k_half,
                           uint32_t iters, uint64_t seed, uint32_t mode, const uint32_t* train,
                           uint64_t n_train, unsigned threads, so_index** out);
/* index.cpp:147-170 (two-call: buf == NULL -> size only) */
int so_serialize_index(const so_index* idx, unsigned char* buf, uint64_t cap, uint64_t* len);
/* index.cpp:191-293 */
int so_deserialize_index(const unsigned char* bytes, uint64_t len, so_index** out);
void so_index_free(so_index* idx);
int so_index_info(const so_index* idx, uint64_t* n, uint32_t* d, uint32_t* ns, uint32_t* k_half);

/* query.cpp:42-64 */
int so_centroid_distances(const float* half_query, uint32_t dim, const float* centroids,
                          uint32_t k_half, double* dists, uint32_t* order);
/* query.cpp:66-121 (kind 0) and tests/support/oracles.cpp:63-88 (kind 2) */
int so_traverse(int kind, double alpha, uint64_t n, const double* d1, const uint32_t* o1,
                const double* d2, const uint32_t* o2, uint32_t k_half, const uint64_t* offsets,
                uint32_t* c1, uint32_t* c2, uint64_t* cum, double* sums, uint64_t cap,
                uint64_t* count);
/* query.cpp:159-197 */
int so_rerank(const float* data, uint64_t n, uint32_t d, const float* query, uint32_t qlen,
              const uint32_t* cands, uint64_t m, uint32_t k, uint32_t* ids, double* dists,
              uint32_t* count);
/* query.cpp:199-262, batched like suco_cli.cpp:95-114 */
int so_knn_query_batch(const so_index* idx, const float* data, uint64_t n, uint32_t d,
                       const float* queries, uint64_t nq, uint32_t qlen, double alpha, double beta,
                       uint32_t k, unsigned threads, uint32_t* ids, double* dists,
                       uint32_t* counts, double* wall_s);
/* intermediates of one knn_query: scores (n u32), candidate set ascending (m u32) */
int so_query_intermediates(const so_index* idx, const float* data, uint64_t n, uint32_t d,
                           const float* query, uint32_t qlen, double alpha, double beta, uint32_t k,
                           uint32_t* scores, uint32_t* cands, uint64_t* m_out,
                           uint32_t* cells_per_subspace, uint64_t* cumulative);

#ifdef __cplusplus
}
#endif
#endif
