// pattern.h -- device-resident analysis of one sparsity pattern (internal).
#pragma once
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

namespace npcg {

// One direction (forward = lower rows ascending, backward = upper rows
// descending) of the chunked triangular-solve schedule.
//
// Rows are split into `chunks` contiguous ranges; inside a chunk rows are
// grouped by chunk-local level (longest chain of intra-chunk dependencies).
// A CTA owning a (chunk, batch-column group) unit walks its levels with one
// __syncthreads per level and keeps the last `window` levels of solved
// values in a shared-memory ring. Values from earlier chunks are read from
// global memory: every solved value is published with a relaxed store over
// a sentinel NaN, so a consumer simply polls the value itself -- no fences,
// no counters (kernels.cu).
//
// All per-entry data is stored in schedule order, so the entries of one
// level are one contiguous block that can be prefetched into L1 a few
// levels ahead of use.
struct Schedule {
    int32_t chunks = 0;       // number of chunks (processing order)
    int32_t chunk_rows = 0;   // rows per chunk (last may be short)
    int32_t window = 1;       // ring depth in levels
    int32_t maxw = 1;         // max rows in one chunk-local level
    int32_t total_levels = 0; // sum over chunks of their level counts
    int32_t max_chunk_levels = 0;
    int32_t levels_global = 0;
    int64_t entries = 0;          // strict-triangle entries (= nnz_lower)
    int64_t padded_entries = 0;   // factor-value slots (levels padded to even counts)
    int32_t max_words = 0;        // largest packed level block (int32 words)
    int32_t max_se = 0;           // largest padded entry count of a level
    int32_t maxx = 0;             // most foreign dependencies in one level
    // device arrays (see pattern.cpp build_direction for the packed layout)
    int32_t *packed = nullptr;    // per-level blocks: rows | eoff | dep | xrow
    int32_t *lvl_woff = nullptr;  // [total_levels+1] word offset of each block
    int32_t *lvl_meta = nullptr;  // [total_levels][4] nrow, ne, nx, factor offset
    int32_t *chunk_lvl = nullptr; // [chunks+1] first level of each chunk
    int32_t *sperm = nullptr;     // [padded_entries] CSR position (or -1) of a factor slot
};

struct SchedSet {
    Schedule fwd, bwd;
    ~SchedSet();
};

// Line-wavefront schedule (trsv_line.cu): the rows split into "lines",
// maximal runs in which every row depends on its predecessor (grid lines of
// a mesh in natural order). One thread owns one line and walks its rows in
// solve order; step s of the CTA solves every row whose level is s, so the
// in-line dependency stays in a register and the cross-line ones are read
// from a per-line shared-memory ring of the last `window` values.
// Per (step, thread) the schedule stores MD dependency descriptors and the
// matching factor slots, step-major: desc[step][e][T] (int16) with
//   -1 = previous row of the line, >= 0 = ring slot, zslot = padding,
//   desc[.][0] = kNoRow when the thread has no row at that step,
// and vperm[step][e][T] = CSR position of the factor value (-1 = padding).
// Only built when the whole pattern fits one CTA (lines <= 1024, window <= 16).
constexpr int32_t kLineBatch = 6;          // steps staged per batch
constexpr int16_t kNoRow = -2;             // desc[.][0]: thread idle at this step

struct LineDir {
    int32_t nlines = 0, T = 0, steps = 0, steps_pad = 0, window = 1, md = 1, zslot = 0;
    int32_t *line_row0 = nullptr;  // [T] first row of each thread in solve order (-1: idle)
    int32_t *line_len = nullptr;   // [T] rows of each thread's line
    int16_t *desc = nullptr;       // [steps_pad][md][T]
    int32_t *vperm = nullptr;      // [steps_pad][md][T]
};
struct LineSched {
    bool ok = false;
    LineDir fwd, bwd;
    ~LineSched();
};

struct Pattern {
    int64_t n = 0, nnz = 0, nnz_lower = 0;
    bool full_diag = false, symmetric = false, factor_ok = false;
    std::vector<int32_t> h_rp, h_col, h_dp, h_pair;
    int32_t *rp = nullptr, *col = nullptr, *dp = nullptr, *pair = nullptr;
    int32_t *lower_slot = nullptr; // [nnz_lower] CSR position of each strict-lower entry
    int32_t *src = nullptr;        // [nnz] row of each stored entry (edge source, gnn.py:83)
    std::map<int32_t, std::unique_ptr<SchedSet>> scheds;  // by chunk rows
    std::unique_ptr<LineSched> lines;                      // built on first use
    std::mutex mu;
    ~Pattern();
    // Schedule for `chunk_rows` (built on first use); nullptr + err on failure.
    SchedSet *schedule(int32_t chunk_rows, std::string &err);
    // Line schedule, or nullptr when the pattern does not qualify.
    LineSched *line_schedule();
};

// Rows per chunk for a solve over B columns in groups of G (heuristic,
// overridable with NPCG_CHUNK_ROWS).
int32_t choose_chunk_rows(int64_t n, int B, int G);

}  // namespace npcg
