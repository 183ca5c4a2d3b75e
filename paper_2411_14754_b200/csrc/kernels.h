// Launch interfaces of the query-path and build-path kernels (host side).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace suco_gpu {

// ---------------------------------------------------------------- traverse
// One warp per (query, subspace): project the query halves, exact fp64
// centroid distances + (dist, id) ranking (query.cpp:42-64), then Dynamic
// Activation (query.cpp:66-121) until the cumulative global cell size
// reaches `target` = collision_count(alpha, n). Emits retrieved cell indices
// (c1 * k_half + c2) in retrieval order.
struct TraverseArgs {
    const float* queries;  // nq x d
    uint32_t d;
    uint64_t nq;
    const uint32_t* dims;  // concatenated layout dims
    const SubDesc* sub;    // ns
    const float* cent;     // concatenated centroids
    const uint32_t* cell_size;  // ns x K
    uint32_t ns, k_half, K, hmax;
    uint64_t target;
    uint32_t* cells;   // nq x ns x K
    uint32_t* ncells;  // nq x ns
    double* dbg_sum;   // optional, nq x ns x K
    uint64_t* dbg_cum; // optional, nq x ns x K
    unsigned long long* stat_cum;  // optional: += final cumulative of every traversal
    char mode;         // Tuning::traverse (0 = by shape)
    uint32_t cs_global;  // set by launch_traverse: the merge kernel reads cell sizes from global memory
};
cudaError_t launch_traverse(const TraverseArgs& a, cudaStream_t st);
uint32_t traverse_launch_count(const TraverseArgs& a);  // kernels launch_traverse issues (1, or 2: rank + merge)

// Stand-alone stages for parity tests.
cudaError_t launch_centroid_distances(const float* d_q, uint32_t dim, const float* d_cent, uint32_t k_half,
                                      double* d_dists, uint32_t* d_order, cudaStream_t st);
cudaError_t launch_da_only(const double* d1, const uint32_t* o1, const double* d2, const uint32_t* o2,
                           uint32_t k_half, const uint32_t* cell_size, uint64_t target, uint32_t* cells,
                           uint32_t* ncells, double* sums, uint64_t* cum, cudaStream_t st);

// ------------------------------------------------------------------ select
// Cluster kernel: each cluster of CS CTAs owns one query; CTA r owns id slabs
// r, r+CS, ... of CH ids with u8 collision counters in shared memory.
// Counting (query.cpp:229-239), then the global top-m by (score desc, id asc)
// (query.cpp:242-260) via a per-slab score histogram exchanged over DSMEM, a
// threshold score T and an id-ordered tie quota per slab.
struct SelectArgs {
    const uint32_t* ids;       // ns x n   (IMI ids, ascending within a cell)
    const uint32_t* slab_off;  // ns x K x (nslabs + 1): start of slab j inside each cell
    const uint32_t* cells;     // nq x ns x cells_cap
    const uint32_t* ncells;    // nq x ns
    uint32_t cells_cap;
    uint64_t n;
    uint32_t ns, K, nslabs, CH, rounds, CS;
    uint64_t m;
    uint64_t nq;          // queries in this launch (persistent clusters loop over them)
    uint32_t* cands;      // nq x m (candidate set, unordered)
    uint8_t* scores_dbg;  // optional nq x n
    uint64_t scores_stride;  // row stride of scores_dbg (0 = n); a multiple of 16 enables 16-byte stores
};
struct SelectConfig {
    uint32_t CS, CH, nslabs, rounds;
    size_t smem;
    int clusters;  // resident clusters (persistent grid); 0 = unknown
};
SelectConfig plan_select(uint64_t n, uint32_t ns, int cluster_size);
cudaError_t launch_select(const SelectArgs& a, const SelectConfig& cfg, uint64_t nq, cudaStream_t st);
cudaError_t launch_slab_offsets(const uint32_t* cell_off, const uint32_t* ids, uint64_t n, uint32_t ns,
                                uint32_t K, uint32_t CH, uint32_t nslabs, uint32_t* slab_off,
                                cudaStream_t st);

// ------------------------------------------------------------------ dense select
// Bit-sliced dense selection over 32-query blocks (dense.cu): same output as
// select_kernel (the top-m candidate set, unordered) when N_s <= 8.
struct DenseArgs {
    const uint4* codes;        // n x 8 u16: s*K + cell of the point in subspace s (N_s*K when s >= N_s)
    const uint32_t* cells;     // nq x ns x cells_cap (traversal output), or compact (cells_off)
    const uint32_t* ncells;    // nq x ns
    const uint64_t* cells_off; // optional nq*ns+1 offsets into a compact `cells` (then ncells unused)
    uint32_t cells_cap, ns, K;
    uint64_t n, nq, m;
    uint32_t P, WP;            // pieces of WP consecutive points (one warp each)
    uint16_t* hist;            // nq x P x 8: #score >= t, t = 1..8
    uint32_t* T;               // nq
    uint32_t* quota;           // nq x P
    uint32_t* base;            // nq x P
    uint32_t* base2;           // single pass: nq x P, the offsets of the pieces' ties (base: their score > T entries)
    uint32_t* cands;           // nq x m
    // single-pass (fused) select: a speculative lower bound L on T per query, a superset slot of
    // C entries (in-piece offset << 4 | score, id order) per (query, piece), and a fallback flag
    uint32_t pstride;          // K1 over a sample: hist row j scans piece j * pstride (0 = 1)
    uint16_t* hsample;         // nq x Ps x 8 sampled histograms (K0)
    uint32_t Ps;               // sampled pieces
    uint32_t sWP;              // points per sampled piece (0 = WP): 2048 whatever the single pass's piece size
    uint32_t* L;               // nq
    uint16_t* cbuf;            // single pass: [query][piece][B] in-piece offsets of score >= L (bit 15: > L)
    uint16_t* ccnt;            // single pass: nq x P entries found (may exceed B)
    uint32_t* qflag;           // nq: 1 = fall back to the exact two-pass emission for this query
    uint32_t B;                // single pass: candidate buffer entries per (piece, query), multiple of 8
    uint32_t* h2;              // single pass: nq x P, #score >= L | #score >= L+1 << 16
    uint32_t* qmap;            // fallback emission: block-local query j -> query qmap[q0 + j]
    uint32_t* nmap;            // device count of qmap entries
    uint32_t ppw;                 // fused pass: pieces per warp (set by the launcher)
    uint32_t stage_all;           // fused pass: stage every block's stores (tests; else by density)
    uint32_t half;                // 16-query blocks, u16 masks, codes = cell + 1 per subspace (large N_s*K)
    uint32_t hgroup;              // half-width mode, eight subspaces: interleaved table (slot c' * 8 + s, rotated codes)
    uint32_t nc;                  // uint4 code vectors per point: 1 (N_s <= 8, default) or 2 (N_s <= 16)
    uint32_t* pcut;               // single pass: nq, tie entries are stored only in pieces < pcut[q]
    uint32_t no_cut;              // tests: store every tie (pcut = P)
    uint32_t shG, shR, shPPB;     // shard single pass: G shards, this shard r, pieces per id block (0: unsharded);
                                  // local piece p is global piece ((p / shPPB) * G + r) * shPPB + p % shPPB
    uint32_t* clist;              // single pass: nq x 2 — unflagged queries with dense supersets from the front,
                                  // sparse ones from nq on (compaction work lists, any order)
    uint32_t* nclist;             // their two counts
    uint32_t compact_rows;        // Tuning::dense_compact_rows: grid rows of the warp compaction (0 = 1024)
    uint32_t compact_mode;        // Tuning::dense_compact: 0 by density, 1 thread per piece, 2 warp per (query, piece)
    uint32_t pair;                // half mode: the fused pass as 2-CTA clusters with 32-bit masks of 4 subspaces each
    float cut_scale;              // tie cut = P * need/ties * cut_scale + cut_pad pieces (0: defaults 1.25, 8)
    uint32_t cut_pad;
    uint32_t words;               // Tuning::dense_words (0 = by shape)
    uint8_t* scores_dbg;          // optional (nq == 1): K3 writes query 0's SC-score of every point (parity)
};
// Mask-table slots of the 32-bit dense select. Eight subspaces (every NC = 1 configuration of the
// bench) use a bank-grouped layout: subspace s owns banks 4s..4s+3, slot(s, c) = (c / 4) * 32 +
// 4s + c % 4, and a point's code position j holds subspace (j + p) % 8, so lane l of a tile looks
// up subspace (j + l) % 8 in load j: four lanes per 4-bank group instead of 32 lanes over 32
// banks (expected worst bank load 2.95 instead of 3.53 for random cells). Other subspace counts
// keep slot(s, c) = s * K + c with position j = subspace j. The last slot is the zero slot.
__host__ __device__ inline bool dense_grouped(uint32_t ns) { return ns == 8; }
__host__ __device__ inline uint32_t dense_none(uint32_t ns, uint32_t K) {
    return dense_grouped(ns) ? 8u * ((K + 3u) & ~3u) : ns * K;
}
__host__ __device__ inline uint32_t dense_slot(uint32_t ns, uint32_t K, uint32_t s, uint32_t c) {
    return dense_grouped(ns) ? ((c >> 2) << 5) | (s << 2) | (c & 3u) : s * K + c;
}
bool dense_supported(uint32_t ns, uint32_t K);
// 9..16 subspaces: two code vectors per point, 5 score planes, 16 histogram levels (config 3)
bool dense_wide_supported(uint32_t ns, uint32_t K);
size_t dense_smem(uint32_t ns, uint32_t K);
// Half-width mode for tables too large for 32-bit masks (config 5: N_s*K = 80,000 cells): 16-query
// blocks, one u16 mask per (subspace, cell), two points per lane; codes hold cell + 1 per subspace
// (0 = no cell), n_pad = rows rounded up to whole pieces (padding rows are all 0).
bool dense_half_supported(uint32_t ns, uint32_t K);
// the cluster-pair fused pass for half-mode tables: 5..8 subspaces, 4 x (K + 1) 32-bit slots per CTA
bool dense_pair_supported(uint32_t ns, uint32_t K);
cudaError_t launch_dense_codes_half(const uint32_t* ids, const uint32_t* cell_off, uint64_t n, uint64_t n_pad,
                                    uint32_t ns, uint32_t K, uint16_t* codes, uint32_t group, uint32_t sched_passes,
                                    cudaStream_t st);
cudaError_t launch_dense_codes(const uint32_t* ids, const uint32_t* cell_off, uint64_t n, uint32_t ns, uint32_t K,
                               uint16_t* codes, uint32_t sched_passes, cudaStream_t st);
cudaError_t launch_dense_select(const DenseArgs& a, cudaStream_t st);  // hist + plan + emit
// the single pass's stages (launch_dense_select_fused runs them; the shard protocol interleaves its exchanges)
cudaError_t launch_dense_sample(const DenseArgs& a, cudaStream_t st);
cudaError_t launch_dense_fused_pass(const DenseArgs& a, cudaStream_t st);
cudaError_t launch_dense_compaction(const DenseArgs& a, cudaStream_t st);
// single pass: K0 sample -> L estimate -> fused hist + superset -> plan + checks -> compaction ->
// exact emission for the flagged query blocks (rare); needs hsample/L/cbuf/ccnt/qflag/B
// main_done (optional) is recorded once every unflagged query's candidates are written; the
// flagged queries' fallback then runs on fb_st (optional, else st).
cudaError_t launch_dense_select_fused(const DenseArgs& a, cudaStream_t st, cudaEvent_t main_done = nullptr,
                                      cudaStream_t fb_st = nullptr);
// Shard protocol pieces: K1 alone (+ its histograms as [nq][P][N_s + 2] u32 rows with the
// piece length first, the exchange format) and K3 alone with the globally planned T/quota/base.
cudaError_t launch_dense_hist(const DenseArgs& a, cudaStream_t st);
cudaError_t launch_dense_hist_rows(const DenseArgs& a, uint32_t* out, cudaStream_t st);
cudaError_t launch_dense_emit(const DenseArgs& a, cudaStream_t st);
constexpr uint32_t kDensePiece = 2048;  // points per piece (one warp)
constexpr uint32_t kDenseBuf = 96;      // single-pass candidate buffer entries per 2048 points of a (piece, query)
constexpr uint64_t kQ8MinCands = 8192;  // the int8 screen pays off from this many candidates per query
constexpr uint32_t kDenseCodePad = 128;  // zero-slot code rows past n (the fused pass loads two tiles ahead)
constexpr uint32_t kFusedPiece = 8192;
constexpr uint32_t kMaxPiece = 32768;   // largest single-pass piece (SUCO_DENSE_PIECE): 15-bit in-piece offsets  // points per piece of the single-pass select (half-width mode: kDensePiece)

// ------------------------------------------------------------------ rerank
// Exact fp64 re-rank of the candidate rows (query.cpp:159-197) with a
// warp-level (dist, id) top-k; k > 32 takes a generic selection path.
struct RerankArgs {
    const float* data;  // n x d
    uint64_t n;
    uint32_t d;
    const float* queries;   // nq x d
    const uint32_t* cands;  // nq x m
    uint64_t m;
    uint32_t k;
    uint32_t* out_ids;    // nq x k
    double* out_dists;    // nq x k
    double* all_d;        // generic path scratch nq x m
    uint32_t* all_id;     // generic path scratch nq x m
    float data_int_max;   // >= 0: every data value is an integer with |v| <= this; < 0: not certified
    const uint32_t* counts;  // optional per-query candidate counts (<= m; m is then the row stride)
    bool squared;            // output squared distances (shard-local top-k for the cross-shard merge)
    uint32_t shard_b, shard_G, shard_s; // unused by the kernels: shards re-rank LOCAL rows (local order ==
                                        // global order) and launch_shard_ids maps the k outputs to global ids
    const uint8_t* data8;  // optional u8 copy of the rows (data certified integer in [0, 255]), n x dpad
    uint32_t dpad;         // row bytes of data8 (d rounded up to 16)
    bool identity;         // exact kNN: candidate i of every query is id i (cands unused, m = n)
    const uint32_t* qskip;  // optional: queries with qskip[q] != 0 are left for a later pass
    const uint32_t* qlist;  // optional: re-rank only qlist[0 .. *nlist) (the grid still spans nq)
    const uint32_t* nlist;
    const int8_t* q8;       // optional int8 screen records of float rows (n x qrec), rerank_q8_kernel's input:
                            // qpad int8 values, then {s, |x|^2, ||s a|| (up), ||x - s a|| (up)} (s < 0: no
                            // bounds), padded to a multiple of 64 bytes (the DRAM access granule)
    uint32_t qpad;          // int8 bytes of a record (d rounded up to 16)
    uint32_t qrec;          // record stride (qpad + 16 rounded up to 64)
    uint32_t qpre;          // prefix-bound layout: prefix words (16 dims each; 0 = plain records)
    uint64_t q8_min;        // candidates per query from which the int8 screen is used (kQ8MinCands; tests: 0)
    uint32_t qsplit;        // prefix-bound layout: bytes of a record's prefix part (stride of the prefix array)
    const int8_t* q8b;      // prefix-bound layout: the rests of the records (q8 + rows * qsplit), stride qrec - qsplit
    bool no_tma;            // !Tuning::rerank_tma: 16-byte cp.async row gathers instead of per-row TMA bulk copies
    unsigned long long* screen_stats;  // optional diagnostics: [0] += exact re-ranks, [1] += queries re-ranked in full
    bool u8_regs;           // Tuning::rerank_u8_regs: the register byte kernel instead of the smem ring
    uint8_t pipe;           // 0: certified fp32 screen (default), 1: pipelined fp64, 2: unpipelined
};
cudaError_t launch_rerank(const RerankArgs& a, uint64_t nq, cudaStream_t st);

// ------------------------------------------------------------------- shards
// ids[i] = ((l / b) * G + shard) * b + l % b for the n local ids l (0xffffffff kept).
cudaError_t launch_shard_ids(uint32_t* ids, uint64_t n, uint32_t b, uint32_t G, uint32_t shard, cudaStream_t st);
// counts == phase A (per-cell owned counts); local_ids != nullptr: phase B (compaction)
cudaError_t launch_shard_imi(const uint32_t* ids, const uint32_t* cell_off, uint64_t n, uint32_t ns, uint32_t K,
                             uint32_t b, uint32_t G, uint32_t shard, uint32_t* counts, const uint32_t* local_off,
                             uint64_t n_local, uint32_t* local_ids, cudaStream_t st);

// The sharded select's plan (dense.cu): per-shard totals #(score >= t) [nq][16];
// from every shard's totals [G][nq][16]: T, need and the per-local-block ties at T [nq][nbl_max];
// from every shard's ties [G][nq][nbl_max]: per-piece quota / base (into a.quota / a.base, a.T
// read) and the local candidate count per query. ppb = pieces per block.
cudaError_t launch_shard_totals(const DenseArgs& a, uint32_t* tot, cudaStream_t st);
// the shard protocol's single pass (dense.cu): sampled totals (nq x 17 u32: #(score >= t), t = 1..16,
// and the points sampled) -> all-reduce -> bound (same L and tie cut on every shard) -> fused pass ->
// per-query #(score > L) and per-block ties -> all-reduce / all-gather -> plan (quotas, offsets, the
// shard's candidate counts, flags; *nflag += flagged queries) -> compaction
cudaError_t launch_shard_sample(const DenseArgs& a, uint32_t* sum17, cudaStream_t st);
cudaError_t launch_shard_bound(const DenseArgs& a, const uint32_t* sum17, uint64_t n_global, uint32_t P_global,
                               cudaStream_t st);
cudaError_t launch_shard_fused_sums(const DenseArgs& a, uint32_t ppb, uint32_t nbl, uint32_t nbl_max, uint32_t* gt,
                                    uint32_t* ties, cudaStream_t st);
cudaError_t launch_shard_fused_plan(const DenseArgs& a, const uint32_t* gt_sum, const uint32_t* gt_local,
                                    const uint32_t* ties_all, uint32_t G, uint32_t shard, uint64_t nb_global,
                                    uint32_t ppb, uint32_t nbl, uint32_t nbl_max, uint32_t* qblk, uint32_t* counts,
                                    uint32_t* nflag, cudaStream_t st);
cudaError_t launch_shard_ties(const DenseArgs& a, const uint32_t* tot_all, uint32_t G, uint32_t ppb, uint32_t nbl,
                              uint32_t nbl_max, uint32_t* T, uint64_t* need, uint32_t* ties, cudaStream_t st);
cudaError_t launch_shard_quota(const DenseArgs& a, const uint32_t* ties_all, uint32_t G, uint32_t shard,
                               uint64_t nb_global, uint32_t ppb, uint32_t nbl, uint32_t nbl_max, const uint64_t* need,
                               uint32_t* qblk, uint32_t* counts, cudaStream_t st);
// k smallest (squared distance, id) over G ascending local lists [G][nq][k], sqrt -> out [nq][k]
cudaError_t launch_merge_topk(const uint32_t* ids_all, const double* sq_all, uint32_t G, uint64_t nq, uint32_t k,
                              uint32_t* out_ids, double* out_d, cudaStream_t st);
// out[i] = sum over g of rows[g][i] (the in-process communicator's all-reduce)
cudaError_t launch_sum_rows_u32(const uint32_t* rows, uint32_t G, uint64_t count, uint32_t* out, cudaStream_t st);

// ------------------------------------------------------------------- build
cudaError_t launch_cell_sizes(const uint32_t* cell_off, uint32_t ns, uint32_t K, uint32_t* cell_size,
                              cudaStream_t st);
cudaError_t launch_check_finite(const float* data, uint64_t count, int* flag, cudaStream_t st);
// out2[0] |= 1 if any value is non-integral; out2[1] = max |value| as float bits (both pre-zeroed)
// out3[0] |= 1 non-integer, out3[1] = max |v| bits, out3[2] |= 1 negative (zero out3 first)
cudaError_t launch_int_stats(const float* data, uint64_t count, unsigned int* out3, cudaStream_t st);
cudaError_t launch_pack_u8(const float* data, uint64_t n, uint32_t d, uint32_t dpad, uint8_t* out, cudaStream_t st);
// int8 screen records of float rows: n x qrec bytes (see RerankArgs::q8)
cudaError_t launch_pack_q8(const float* data, uint64_t n, uint32_t d, uint32_t qpad, uint32_t qrec, uint32_t qpre,
                           uint32_t qsplit, int8_t* out,
                           cudaStream_t st);

// SC-Linear (sclinear.cu): exact per-subspace distances, top-c per (query, subspace) by a radix
// select with id-ordered ties, scores, then the m candidates; batches of B queries.
struct ScArgs {
    const float* data;             // n x d rows
    uint64_t n;
    uint32_t d, ns;
    const uint32_t* dims;          // concatenated whole-subspace dims (layout order)
    const uint32_t* sub_off;       // ns + 1 prefix offsets into dims
    const uint8_t* consec;         // ns: dims form one consecutive run -> sq_euclidean_raw
    const float* q;                // B queries, d floats each
    unsigned long long* keys;      // (set by launch_sc_batch) B x n distance bit patterns of one subspace
    void* scratch;                 // sc_batch_bytes(n, B, m)
};
size_t sc_batch_bytes(uint64_t n, uint32_t B, uint64_t m);
// scores_out (optional, B x n u8): the SC-scores; cands (optional, B x m): the candidate sets
cudaError_t launch_sc_batch(ScArgs a, uint32_t B, uint64_t c, uint64_t m, uint32_t* cands, uint8_t* scores_out,
                            cudaStream_t st);

}  // namespace suco_gpu
