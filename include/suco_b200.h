/*
 * suco_b200.h — the drop-in C-ABI boundary of the B200-native SuCo hot path.
 *
 * Plain C, plain pointers and sizes, no exceptions and no torch types. Every
 * entry point names the reference interface (/root/reference/proj) it
 * replaces; INTEGRATION.md shows the binding a maintainer adds on the
 * reference side. The C++ mirror of the reference API (typed exceptions,
 * suco::gpu namespace) is include/suco_b200.hpp; the Python mirror is the
 * paper_2411_14754_b200 package. All compute runs on the GPU: there is no
 * CPU fallback — without a usable CUDA device every compute call returns
 * SUCO_ERR_INTERNAL with a message.
 *
 * Status codes mirror the reference's exception taxonomy (error.hpp:9-37)
 * and the CLI exit codes (suco_cli.cpp:693-707):
 */
#ifndef SUCO_B200_H
#define SUCO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SUCO_OK 0
#define SUCO_ERR_INTERNAL 1       /* suco::Error / CUDA / NCCL failure                  */
#define SUCO_ERR_CONFIG 2         /* suco::ConfigError                                  */
#define SUCO_ERR_FORMAT 3         /* suco::FormatError (vecs files, io.cpp:20-84)       */
#define SUCO_ERR_INCOMPATIBLE 4   /* suco::IncompatibilityError                         */
#define SUCO_ERR_CONTRACT 5       /* suco::ContractError                                */
#define SUCO_ERR_CORRUPT_INDEX 6  /* suco::CorruptIndexError (a FormatError; index     */
                                  /* bytes, index.cpp:191-293); CLI exit code 3 as well */

/* IndexParams (index.hpp:53-61). mode: 0 Contiguous, 1 Shuffled (subspace.hpp:13-16). */
typedef struct suco_index_params {
    uint32_t num_subspaces; /* default 8  */
    uint32_t k_half;        /* default 50 */
    uint32_t iterations;    /* default 10 */
    uint32_t mode;          /* default 0  */
    uint64_t seed;          /* default 42 */
} suco_index_params;

/* CollisionParams (sc_linear.hpp:22-31). */
typedef struct suco_collision_params {
    double alpha; /* default 0.05  */
    double beta;  /* default 0.005 */
    uint32_t k;   /* default 50    */
} suco_collision_params;

/* Opaque device-resident index: layout, centroids, IMI and the dataset rows
 * (the reference index holds no dataset, index.hpp:63-66; the GPU index must
 * own device copies of the rows it re-ranks). Immutable after build/load:
 * like the reference's (index.hpp:63-66), any number of threads may query
 * one index at once. */
typedef struct suco_gpu_index suco_gpu_index;

/* Per-call query state — the reference's caller-owned QueryScratch
 * (query.hpp:72-78): pipeline scratch, its CUDA streams and events, and the
 * profiling counters of the last call. Bound to the index it was created
 * for; one thread at a time. Query calls given NULL borrow a context from
 * the index's internal pool. */
typedef struct suco_gpu_query_ctx suco_gpu_query_ctx;

/* Communicator of the multi-GPU shard protocol (one rank per GPU). */
typedef struct suco_comm suco_comm;

/* Message of the last failing call on this thread. */
const char* suco_last_error(void);

/* Number of visible CUDA devices (0 on a CPU-only host). */
int suco_gpu_device_count(int* count);

/* ---------------------------------------------------------------- params
 * collision_count (sc_linear.hpp:36, sc_linear.cpp:39-42),
 * candidate_count (sc_linear.hpp:40, sc_linear.cpp:44-47),
 * CollisionParams::validate (sc_linear.hpp:30, sc_linear.cpp:26-37). Host
 * arithmetic, bit-identical to the reference's snapping rule. */
uint64_t suco_collision_count(double alpha, uint64_t n);
uint64_t suco_candidate_count(double beta, uint64_t n, uint64_t k);
int suco_validate_collision_params(const suco_collision_params* p, uint64_t n);

/* ----------------------------------------------------------------- build
 * build_index (index.hpp:85, index.cpp:98-145) on `device`. Checks the
 * Dataset invariants (core.cpp:8-21 -> CONTRACT) then the reference's order:
 * k_half/iterations/n<k_half -> CONFIG, n > 2^32-1 -> CONTRACT, layout ->
 * CONFIG. Output is identical to the reference's build for the same input. */
int suco_gpu_build_index(const float* data, uint64_t n, uint32_t d, const suco_index_params* params,
                         int device, suco_gpu_index** out);

/* Config 5's sampled build (BASELINE.json configs[4]: "centroids trained on a seeded 1% sample").
 * The reference has no API for it; this composes the reference's own steps: the 2*N_s k-means
 * jobs of build_index (index.cpp:120-137, kmeans.cpp:118-194, seeds derive_seed(seed, job)) run
 * on the rows train_ids[0..n_train) only (strictly ascending, in that order), then EVERY row is
 * assigned to its nearest centroid by kmeans.cpp:19-33's rule (fp64, strict '<') and build_imi
 * (index.cpp:69-96) runs over all n. train_ids = 0..n-1 gives exactly suco_gpu_build_index.
 * Checks: as suco_gpu_build_index with n_train in place of n for the k_half test (CONFIG), then
 * ids not strictly ascending or >= n -> CONTRACT. The result serializes like any index (the
 * `.suco` format has no sample field) and the reference's load_index/knn_query accept it.
 * For both build entry points `data` may be host memory or device memory on `device`. */
int suco_gpu_build_index_sampled(const float* data, uint64_t n, uint32_t d, const suco_index_params* params,
                                 const uint32_t* train_ids, uint64_t n_train, int device, suco_gpu_index** out);

/* deserialize_index (index.hpp:107, index.cpp:191-293) + check_compatible
 * (index.hpp:108, index.cpp:295-305): uploads a serialized `.suco` index and
 * the dataset it was built from. Corrupt bytes -> CORRUPT_INDEX naming the section;
 * (n, d) mismatch -> INCOMPATIBLE. */
int suco_gpu_load_index(const unsigned char* bytes, uint64_t len, const float* data, uint64_t n, uint32_t d,
                        int device, suco_gpu_index** out);

/* serialize_index (index.hpp:99, index.cpp:147-170): byte-identical to the
 * reference's serialization of the same index. Two-call protocol: with
 * buf == NULL only *len is written. */
int suco_gpu_serialize_index(const suco_gpu_index* index, unsigned char* buf, uint64_t cap, uint64_t* len);

/* Host copies of one subspace's codebook (SubspaceCodebook, index.hpp:44-50):
 * centroids_first k_half x h1, centroids_second k_half x h2, IMI offsets
 * (k_half^2 + 1, u64) and ids (n, u32). Any pointer may be NULL. */
int suco_gpu_index_subspace(const suco_gpu_index* index, uint32_t subspace, float* centroids_first,
                            float* centroids_second, uint64_t* imi_offsets, uint32_t* imi_ids);

/* n, d, params and the per-subspace layout (SubspaceLayout, subspace.hpp:27-50):
 * dims (d entries, concatenated in subspace order), sizes (N_s), half_split (N_s).
 * Layout pointers may be NULL. */
int suco_gpu_index_info(const suco_gpu_index* index, uint64_t* n, uint32_t* d, suco_index_params* params,
                        uint32_t* dims, uint32_t* sizes, uint32_t* half_split);

void suco_gpu_free_index(suco_gpu_index* index);

/* ----------------------------------------------------------------- query
 * knn_query (query.hpp:93-96, query.cpp:199-262) over a batch of queries, the
 * way run_suco_batch (suco_cli.cpp:95-114) drives it: results[q] =
 * knn_query(index, dataset, queries[q], params). Check order per the
 * reference: query length != d -> CONTRACT, params -> CONFIG, then null
 * buffers (nq > 0) -> CONTRACT. Outputs are nq x k: ids ascending by
 * (distance, id), distances = sqrt of the fp64 squared distance,
 * bit-identical to the reference. Host buffers; returns when the results are
 * written. `scratch` (may be NULL) is the caller's query context, as the
 * reference's optional QueryScratch* (query.hpp:96). */
int suco_gpu_knn_query_batch(const suco_gpu_index* index, const float* queries, uint64_t nq, uint32_t qlen,
                             const suco_collision_params* params, uint32_t* ids, double* dists,
                             suco_gpu_query_ctx* scratch);

/* Same, with device-resident queries/outputs, enqueued on `stream`
 * (cudaStream_t; NULL = the context's own stream — pass cudaStreamLegacy to
 * order with the legacy default stream). Returns once enqueued. */
int suco_gpu_knn_query_batch_device(const suco_gpu_index* index, const float* d_queries, uint64_t nq, uint32_t qlen,
                                    const suco_collision_params* params, uint32_t* d_ids, double* d_dists,
                                    void* stream, suco_gpu_query_ctx* scratch);

/* Query contexts. create: on the index's device. synchronize: waits for all
 * work the context enqueued. */
int suco_gpu_query_ctx_create(const suco_gpu_index* index, suco_gpu_query_ctx** out);
void suco_gpu_query_ctx_free(suco_gpu_query_ctx* ctx);
int suco_gpu_query_ctx_synchronize(suco_gpu_query_ctx* ctx);

/* Stage profiling: when enabled, every query call through this context
 * records CUDA events around each kernel; suco_gpu_query_ctx_stage_times
 * then returns the summed device milliseconds of the last call per stage
 * (0 traverse, 1 select, 2 rerank) and the algorithmic work counters of that
 * call: stats[0] = sum over queries and subspaces of the retrieved ids (the
 * final cumulative of every traversal, query.cpp:105-106), stats[1] =
 * queries, stats[2] = m. last_launches: CUDA kernels the last call enqueued
 * (all of them this library's own sm_100a kernels). exchange_bytes: bytes
 * this rank sent through the communicator in the last shard query. */
int suco_gpu_query_ctx_set_profiling(suco_gpu_query_ctx* ctx, int enabled);
int suco_gpu_query_ctx_stage_times(suco_gpu_query_ctx* ctx, double* ms /*3*/, uint64_t* stats /*3*/);
int suco_gpu_query_ctx_last_launches(const suco_gpu_query_ctx* ctx, uint64_t* launches);
int suco_gpu_query_ctx_exchange_bytes(const suco_gpu_query_ctx* ctx, uint64_t* bytes);

/* Per-query intermediates of knn_query for parity checks, from the
 * production kernels: SC-scores (n u32, query.cpp:235-239, as the select
 * stage scored them), the top-m candidate set sorted ascending (m u32,
 * query.cpp:242-260), per-subspace retrieved-cell counts and final
 * cumulative (query.cpp:229-233). scores / cells / cumulative may be NULL. */
int suco_gpu_query_intermediates(const suco_gpu_index* index, const float* query, uint32_t qlen,
                                 const suco_collision_params* params, uint32_t* scores, uint32_t* cands,
                                 uint64_t* m, uint32_t* cells_per_subspace, uint64_t* cumulative);

/* ------------------------------------------------- multi-GPU shard protocol
 * The reference runs on one host (no distributed API); this is the sharded
 * form of build_index / knn_query, bit-identical to them for
 * any number of shards. Points are split block-cyclically: global block j =
 * ids [j*block, (j+1)*block) belongs to shard j % G (block: a multiple of
 * 2048). Every shard keeps the layout, all centroids and the GLOBAL cell
 * sizes, so its traversal makes the global Dynamic-Activation cut; it scores
 * and re-ranks only its own points. A query batch costs three all-gathers:
 * per-shard score totals (-> the global threshold T), per-block tie counts at
 * T (-> each block's tie quota in global id order), and the local top-k
 * (-> a G-way merge by (distance, id)).
 *
 * Communicators: NCCL (one process per GPU: rank 0 makes an id, every rank
 * receives it out of band and creates its member), or in-process (G members
 * driven by G host threads — e.g. G shards on one GPU for tests). Every rank
 * must make the same sequence of shard calls with the same arguments. */
#define SUCO_NCCL_ID_BYTES 128
int suco_comm_nccl_id(unsigned char* id /* SUCO_NCCL_ID_BYTES */);
int suco_comm_nccl_create(const unsigned char* id, int nranks, int rank, int device, suco_comm** out);
int suco_comm_local_create(int nranks, suco_comm** members /* nranks */);
int suco_comm_info(const suco_comm* comm, int* rank, int* size, uint64_t* bytes_sent);
void suco_comm_free(suco_comm* comm);

/* Block size for n points over num_shards shards: a power of two in
 * [2048, 65536], about n / (100 * num_shards), so the tie quota (the lowest
 * ids at the threshold score) spreads over >= 16 block rounds of shards. */
int suco_gpu_shard_block_hint(uint64_t n, uint32_t num_shards, uint32_t* block);

/* build_index (index.cpp:98-145) across the communicator's ranks, each
 * holding only its own rows: `rows` = the rows of global blocks j = rank
 * (mod G), back to back in id order (n_local x d, host or device memory).
 * The 2*N_s k-means jobs run one per rank (job j on rank j % G) on its
 * projected column gathered in global id order — all rows, or the sampled
 * build's ascending train_ids (NULL: all); the centroids are broadcast, each
 * rank assigns its own rows (kmeans.cpp:19-33) and builds its local IMI, and
 * the per-cell counts are all-reduced. The result equals
 * suco_gpu_make_shard(suco_gpu_build_index[_sampled](all rows), rank, G,
 * block). Checks as suco_gpu_build_index (a failure on any rank fails every
 * rank). */
int suco_gpu_build_shard(const float* rows, uint64_t n_global, uint32_t d, const suco_index_params* params,
                         uint32_t block, const uint32_t* train_ids, uint64_t n_train, suco_comm* comm, int device,
                         suco_gpu_index** out);
/* Cut shard `shard` of num_shards from a full index on the same device. */
int suco_gpu_make_shard(const suco_gpu_index* full, uint32_t shard, uint32_t num_shards, uint32_t block,
                        suco_gpu_index** out);
int suco_gpu_shard_info(const suco_gpu_index* index, uint64_t* n_global, uint64_t* n_local, uint32_t* block,
                        uint32_t* shard, uint32_t* num_shards);
/* knn_query over a batch on every rank at once: every rank passes the same
 * queries and parameters and receives the full nq x k result (as
 * suco_gpu_knn_query_batch). The communicator's rank must hold the index's
 * shard. Host-buffer and device-buffer (enqueued on `stream`) forms. */
int suco_gpu_shard_knn_query_batch(const suco_gpu_index* shard, suco_comm* comm, const float* queries, uint64_t nq,
                                   uint32_t qlen, const suco_collision_params* params, uint32_t* ids, double* dists,
                                   suco_gpu_query_ctx* scratch);
int suco_gpu_shard_knn_query_batch_device(const suco_gpu_index* shard, suco_comm* comm, const float* d_queries,
                                          uint64_t nq, uint32_t qlen, const suco_collision_params* params,
                                          uint32_t* d_ids, double* d_dists, void* stream,
                                          suco_gpu_query_ctx* scratch);

/* ------------------------------------------------------------ evaluation
 * exact_knn (eval.hpp:29, eval.cpp:28-62) over a batch, on the index's device
 * copy of the dataset: the k nearest ids by exact fp64 squared distance (the
 * reference's 4-accumulator kernel, or its exact integer equal for u8 data),
 * ties by id, distances = sqrt. k < 1, k > n or a wrong query length ->
 * CONTRACT. Host buffers: queries nq x qlen, ids / dists nq x k. The GPU
 * ground truth of SURVEY §8(f)2; recall/MRE are host arithmetic
 * (paper_2411_14754_b200.recall / mre, eval.cpp:64-102). */
int suco_gpu_exact_knn_batch(const suco_gpu_index* index, const float* queries, uint64_t nq, uint32_t qlen, uint32_t k,
                             uint32_t* ids, double* dists);

/* ------------------------------------------------------------- SC-Linear
 * compute_sc_scores (sc_linear.hpp:45-50, sc_linear.cpp:49-93): for one
 * query, scores[i] = the number of subspaces in which point i is among the
 * collision_count(alpha, n) nearest by exact fp64 distance of the whole
 * subspace projection, ties by id. Uses the reference's two distance orders
 * (sq_euclidean_raw for a consecutive subspace, sq_euclidean_projected
 * otherwise), so the tally is identical. Wrong query length -> CONTRACT;
 * alpha outside (0, 1] -> CONFIG. scores: n host u32s. */
int suco_gpu_sc_scores(const suco_gpu_index* index, const float* query, uint32_t qlen, double alpha, uint32_t* scores);

/* sc_linear_query (sc_linear.hpp:52-53, sc_linear.cpp:95-121) over a batch:
 * the candidate_count(beta, n, k) best points by (score desc, id asc),
 * re-ranked exactly like knn_query. Params are validated first (CONFIG), then
 * the query length (CONTRACT). Host buffers: queries nq x qlen, ids / dists
 * nq x k. The index-free quality baseline of SURVEY §8(f)4. */
int suco_gpu_sc_linear_batch(const suco_gpu_index* index, const float* queries, uint64_t nq, uint32_t qlen,
                             const suco_collision_params* params, uint32_t* ids, double* dists);

/* ------------------------------------------------------------- vecs I/O
 * read_vecs / write_vecs (io.hpp:22-40, io.cpp:99-160): kind 0 = fvecs
 * (f32), 1 = bvecs (u8), 2 = ivecs (i32, |v| <= 2^24). Records parse in
 * order with the reference's checks and messages (FORMAT: open failure,
 * empty file, invalid or inconsistent dim naming the record, truncation
 * naming the byte offset, non-finite f32, ivecs beyond 2^24); at most `limit`
 * records (UINT64_MAX: all; 0: none, a FORMAT error like the reference's).
 * suco_read_vecs fills `out` (cap_rows rows) or, with out == NULL, only
 * reports n and d. */
int suco_read_vecs(const char* path, int kind, uint64_t limit, float* out, uint64_t cap_rows, uint64_t* n, uint32_t* d);
int suco_write_vecs(const char* path, int kind, uint64_t n, uint32_t d, const float* values);
/* Device upload straight from a vecs file: the file streams
 * through two pinned 32 MB stages into the index's device rows (parse of one
 * chunk overlaps the copy of the previous), then build / load as
 * suco_gpu_build_index / suco_gpu_load_index — the host never holds the
 * float matrix. */
int suco_gpu_build_index_from_vecs(const char* path, int kind, uint64_t limit, const suco_index_params* params,
                                   int device, suco_gpu_index** out);
int suco_gpu_load_index_from_vecs(const unsigned char* bytes, uint64_t len, const char* path, int kind, uint64_t limit,
                                  int device, suco_gpu_index** out);

/* ------------------------------------------------ stage-level entry points
 * Each runs the device kernel of one stage on host inputs (parity tests of
 * the reference's free functions). */

/* centroid_distances (query.hpp:27-28, query.cpp:42-64). */
int suco_gpu_centroid_distances(const float* half_query, uint32_t dim, const float* centroids, uint32_t k_half,
                                double* dists, uint32_t* order);

/* dynamic_activation (query.hpp:57-58, query.cpp:66-121) over an IMI given
 * by its CSR offsets (k_half^2 + 1). Writes up to `cap` cells (c1, c2,
 * cumulative, sum_dist) in retrieval order; *count = cells retrieved. */
int suco_gpu_dynamic_activation(double alpha, uint64_t n, const double* dists1, const uint32_t* order1,
                                const double* dists2, const uint32_t* order2, uint32_t k_half,
                                const uint64_t* imi_offsets, uint32_t* c1, uint32_t* c2, uint64_t* cumulative,
                                double* sum_dist, uint64_t cap, uint64_t* count);

/* rerank (query.hpp:83-84, query.cpp:159-197). */
int suco_gpu_rerank(const float* data, uint64_t n, uint32_t d, const float* query, uint32_t qlen,
                    const uint32_t* candidates, uint64_t m, uint32_t k, uint32_t* ids, double* dists);

/* kmeans (kmeans.hpp:46-48, kmeans.cpp:118-194): centroids k x dim,
 * assignments n, repaired cluster ids (<= k * iterations entries). */
int suco_gpu_kmeans(const float* points, uint64_t n, uint32_t dim, uint32_t k, uint32_t iterations,
                    uint64_t seed, int device, float* centroids, uint32_t* assignments, uint32_t* repaired,
                    uint32_t* num_repaired);

/* build_imi (index.hpp:38-39, index.cpp:69-96). */
int suco_gpu_build_imi(const uint32_t* first, const uint32_t* second, uint64_t n, uint32_t k_half,
                       uint64_t* offsets, uint32_t* ids);

#ifdef __cplusplus
}
#endif
#endif /* SUCO_B200_H */
