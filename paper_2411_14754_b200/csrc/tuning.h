// Algorithm choices of the library that tests and A/B runs may override.
//
// Read ONCE — from SUCO_* environment variables — when an index handle is
// created (build / load / shard) or when a stand-alone stage entry point is
// called, then immutable: a query call never reads the environment, and two
// queries on one handle always take the same path. Defaults are the
// measured-best production choices (DESIGN.md §5 lists the measurements).
#pragma once

#include <stdint.h>

namespace suco_gpu {

struct Tuning {
    int cluster = 0;             // SUCO_CLUSTER: cluster-counting select cluster size (0 = by occupancy)
    bool no_u8 = false;          // SUCO_NO_U8: never keep a byte copy of u8-valued rows
    int q8 = 1;                  // SUCO_Q8: int8 screen copy of float rows: 0 none (the fp32 screen reads f32 rows),
                                 // 1 used from kQ8MinCands candidates per query, 2 always (tests)
    uint32_t q8_prefix = 3;      // SUCO_Q8_PREFIX: int8 screen prefix words (16 dims each: 3 = one 64-byte read,
                                 // 1 = one 32-byte sector, 0 = no prefix bound). Measured at cfg4: 3 -> 2,053 of
                                 // 50,000 rows per query past the bound, rerank 7.90 ms; 1 -> 12,600 rows, 8.37 ms
    bool dense = true;           // SUCO_DENSE=0: the cluster-counting select only
    int dense_half = 1;          // SUCO_DENSE_HALF: 0 never, 1 when 32-bit masks do not fit, 2 force
    int dense_pair = 0;          // SUCO_DENSE_PAIR=1: half mode's fused pass on 2-CTA clusters (measured slower at
                                 // cfg5: select 403.6 vs 389.1 ms; half the shared-memory lookups, but the
                                 // per-tile DSMEM exchange costs more than the bank conflicts it saves)
    uint32_t dense_sched = 1;    // SUCO_DENSE_SCHED: local-search passes ordering each point's codes against bank
                                 // conflicts (grouped layout; 0 = the plain lane rotation)
    bool dense_fused = true;     // SUCO_DENSE_FUSED=0: the two-pass dense select
    bool dense_stage = false;    // SUCO_DENSE_STAGE=1: stage every block's stores (tests)
    uint32_t dense_buf = 0;      // SUCO_DENSE_BUF: single-pass buffer entries per (piece, query); 0 = by memory
    float tie_cut_scale = 0.f;   // SUCO_TIE_CUT=scale,pad: tie cut = P * need / ties * scale + pad pieces (A/B; 0: 1.25, 8 x 2048 points)
    uint32_t tie_cut_pad = 0;
    bool dense_nocut = false;    // SUCO_DENSE_NOCUT=1: store every tie (tests)
    uint32_t dense_words = 0;    // SUCO_DENSE_WORDS: mask words per slot (0 auto, 1, 2)
    uint32_t dense_compact = 0;  // SUCO_DENSE_COMPACT: 0 by superset density (default), 1 thread per piece with a
                                 // shared staging copy of the block's output run, 2 warp per (query, piece)
    uint32_t dense_compact_rows = 0;  // SUCO_DENSE_COMPACT_ROWS: grid rows of the warp compaction (A/B)
    uint32_t dense_piece = 0;    // SUCO_DENSE_PIECE: points per piece of the single-pass select (0 = 8192; a
                                 // multiple of 2048 up to 32768; the half-width mode keeps 2048)
    bool dense_stats = false;    // SUCO_DENSE_STATS=1: print the single-pass fallback rate (diagnostics)
    bool rerank_stats = false;   // SUCO_RERANK_STATS=1: print the int8 screen's exact re-rank counts (diagnostics)
    uint32_t tiles = 1;          // SUCO_TILES: minimum pipeline tiles per batch (tests: slot reuse)
    uint64_t scratch_bytes = 0;  // SUCO_SCRATCH_MB: query scratch budget per context (0 = from free memory)
    int fb_overlap = -1;         // SUCO_FB_OVERLAP: overlapped dense fallback (-1 auto, 0, 1)
    char traverse = 0;           // SUCO_TRAVERSE: 0 auto, 'r' rank + merge kernels, 't' one thread kernel, 'w' warp kernel, 's' / 'n' thread kernel with / without split tasks
    bool rerank_u8_regs = false; // SUCO_RERANK_U8_PIPE=0: the register byte re-rank instead of the ring
    bool rerank_tma = false;     // SUCO_RERANK_TMA=1: int8-screen rows by per-row TMA bulk copies (measured slower:
                                 // cfg4 re-rank 12.96 vs 8.58 ms with the warp's coalesced 16-byte cp.async)
    int rerank_pipe = 2;         // SUCO_RERANK_PIPE: 0 unpipelined, 1 pipelined fp64, 2 certified fp32 screen
    bool kpp_serial = false;     // SUCO_KPP_SERIAL=1: k-means++ one-lane serial fold (tests)
    uint64_t build_chunk = 0;    // SUCO_BUILD_CHUNK: rows per assignment chunk of the sampled build (0 = 2 GB)
    uint32_t sc_batch = 0;       // SUCO_SC_BATCH: SC-Linear queries per batch (0 = about 2 GB of keys; tests)
};

Tuning tuning_from_env();

}  // namespace suco_gpu
