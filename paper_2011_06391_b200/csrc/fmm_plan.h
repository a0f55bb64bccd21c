// fmm_plan.h — host-side planning for the device FusedMM path.
//
// Everything here runs once per graph upload (excluded from kernel timing,
// like the paper's preprocessing): the part1d row partition,
// CSR validation, and the per-shard work lists the row kernels consume.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace fmm {

// Edges per chunk when a heavy row is split on the reassociating scheme.
// Chunk boundaries sit at fixed row-relative offsets, so results do not
// depend on the shard count.
// Edges per chunk of a split row: a power of two near total_nnz / 16384,
// clamped to [256, 16384] (2048 for configs 2 and 3, 16384 for config 5). A
// function of the WHOLE graph only, never of a shard, so the chunk
// boundaries — and the results — do not depend on the shard count. Chosen
// for one GPU and eight together (tools/shard_balance.py, r05): config 2
// 1.229 ms / 6.98x at 8 shards with (2048, 128) against 1.186 ms / 3.98x with
// (4096, 512) — one warp folding a 4096-edge row or one lane group a
// 512-edge row floors every shard's kernel at ~0.15-0.3 ms. FMM_CHUNK
// overrides (tuning).
int choose_chunk_edges(int64_t total_nnz);
// Unsplit rows at least this long are folded by a whole warp on the fast
// scheme (a bucket boundary, so they form a prefix of the ordered rows).
// (The threshold is max(64, min(kWideMin, chunk / 16)): rows up to a few
// hundred edges run faster folded by one lane group than spread over a warp
// on one GPU, but a long narrow row floors a small shard's kernel.)
constexpr int kWideMin = 512;
// FMM_WIDE (power of two >= 8, tuning) overrides; read once.
int wide_min(int chunk);
// The threshold the row kernels use depends on d (r3k): a d = 128 row of a
// few hundred edges runs ~5% faster folded by one of the warp's four lane
// groups (the prologue latencies are shared by four rows) than spread over
// the warp, while the eight groups of a d = 32 warp want rows of 128 edges
// up spread. The plan counts the warp-item prefix for every power-of-two
// threshold 64 << k, k < kWideLevels, and the launch picks one by d; the
// rule depends on (chunk, d) only, never on the shard, so results stay
// bitwise independent of the shard count.
constexpr int kWideLevels = 6;  // 64, 128, 256, 512, 1024, 2048
int wide_level_for(int chunk, int d);

struct Int4 {
    int32_t x, y, z, w;
};

// Column bands (r3q). On a graph whose X is far larger than the L2 (config
// 5: 17 GB against 126 MB) a heavy row's gathers mostly miss. When the rows of
// at least `min_deg` edges are cut at fixed COLUMN boundaries (bands of
// `band_cols` columns: 64 MB of d = 256 rows) and the pieces run band by band,
// every warp on the GPU gathers from the same band at the same time, so an X
// row is fetched from DRAM once per band sweep and then served by L2 to every
// heavy row that references it. A piece closes at a band boundary once it has
// `min_len` edges (sparse bands merge forward) and never exceeds the chunk
// size. Rows must have ascending columns (CSR from csr_from_coo has); a row
// that does not falls back to fixed-size chunks. The boundaries depend on the
// row's own columns and on (n, total nnz) only, so results stay bitwise
// independent of the shard count.
struct BandParams {
    int64_t band_cols = 0;  // 0: no banding
    int min_deg = 4096;
    int min_len = 64;
};
// Bands of 65,536 columns when the graph has at least 128 of them; FMM_BANDS=0
// disables, FMM_BAND_COLS / FMM_BAND_MINDEG / FMM_BAND_MINLEN override (tuning).
BandParams choose_bands(int64_t n);

// part1d (kernel.hpp:24-49): boundary i is the smallest row r with
// row_ptr[r]*t >= i*nnz; rows split evenly when nnz == 0. row_ptr may be a
// rebased sub-range (row_ptr[0] subtracted by the caller or not: the rule is
// applied to row_ptr[r] - row_ptr[0]).
std::vector<int64_t> part1d(int64_t m, const int64_t* row_ptr, int t);

// Cost-balanced variant for GPU shards: boundary i is the smallest row r with
// (row_ptr[r] + w*r) * t >= i * (nnz + w*m), i.e. every row also costs w
// edge-equivalents (the per-row work of the row kernels: descriptor, x_u,
// z_u, the first-batch latency). w == 0 is exactly part1d.
std::vector<int64_t> part1d_weighted(int64_t m, const int64_t* row_ptr, int t, double w);

// Validates row_ptr over [row_begin, row_end]: monotone, row_ptr[0] == 0.
// Returns an empty string when valid, else the first violation.
std::string validate_row_ptr(int64_t m, const int64_t* row_ptr);

// Work lists for one shard (rows [row_begin, row_end), local row ids).
struct ShardPlan {
    int64_t row_begin = 0, row_end = 0;   // absolute
    int chunk = 256;                      // edges per chunk of a split row
    int wide = 64;                        // rows with degree >= wide are warp items
    int64_t edge_begin = 0, nnz = 0;      // absolute edge offset, count
    std::vector<int64_t> local_row_ptr;   // rebased, rows+1
    // Rows ordered heavy-first (inside a bucket of degree >= 16 by exact
    // degree): rows with degree > chunk first, then by
    // descending power-of-two degree bucket, stable (natural order) inside a
    // bucket so light rows keep their memory locality.
    std::vector<int32_t> order;
    // items[i] = {order[i], e0 low 32 bits, e0 high 32 bits, degree} with e0
    // the row's first local edge: the kernels read a row's whole descriptor
    // with one 16-byte load
    std::vector<Int4> items;
    int64_t n_split_rows = 0;             // prefix of `order` cut into chunks (degree > chunk, or banded)
    int64_t n_banded_rows = 0;            // of those, cut at column-band boundaries
    int64_t n_wide_rows = 0;              // next rows with degree >= wide
    int64_t n_wide_at[kWideLevels] = {};  // ... with degree >= 64 << k
    std::vector<Int4> chunks;             // {split-row index, first edge (row-relative), edges, slot}, band-major
    std::vector<Int4> split_rows;         // {row, first slot, nchunks, 0}
    int64_t n_slots = 0;
    int64_t nonempty_rows = 0;
    int64_t max_degree = 0;
};

// col_idx (the whole matrix's columns, indexed like row_ptr's edges) is only
// read when bands.band_cols > 0.
ShardPlan build_shard_plan(const int64_t* row_ptr, int64_t row_begin, int64_t row_end, int chunk,
                           const int64_t* col_idx = nullptr, BandParams bands = {});

}  // namespace fmm
