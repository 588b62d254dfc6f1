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
// a mesh in natural order). One thread owns one line; lines are rigid: in
// the forward solve row k of line l is solved at step start[l] + k, and the
// backward solve runs the same steps in reverse. The in-line dependency
// stays in a register, cross-line ones are read from a shared-memory ring
// of every line's last `window` values ([window][T]).
//
// Line order ("slots"): the vectors the solves touch are stored step-major,
// each step holding the contiguous range of lines active at it, so the rows
// of a batch of kLineBatch steps are one contiguous slot range in both
// directions and move with a single bulk copy. Slot ranges of batches are
// padded to multiples of 8 (16-byte aligned copies); padding slots belong to
// no row and hold zeros.
//
// Per batch (in a direction's order) the schedule holds a 16-byte header
// (int32 base[kLineHeader]: slot of line 0 at each step, relative to the
// batch's first slot) followed by [md][slot] int16 descriptors
//   -1 = previous row of the line, >= 0 = ring slot, zslot = padding (zero);
// vperm[md][slot] = CSR position of the matching factor value (-1 = pad).
// Both are structure-of-arrays per batch so a warp's reads are contiguous.
// Only built when the whole pattern fits one CTA (lines <= kLineMaxLines,
// window <= 16, <= 8 dependencies per row) and the pattern is structurally
// symmetric.
constexpr int32_t kLineBatch = 4;      // steps per pipeline stage
constexpr int32_t kLineHeader = 4;     // int32 bases in a batch header (>= kLineBatch; 16 bytes)
constexpr int32_t kLineMaxLines = 512;
constexpr int32_t kLineSlotAlign = 8;  // slots per alignment unit of a batch range

struct LineDir {
    int32_t T = 0, nbatch = 0, window = 1, md = 1, zslot = 0, max_slots = 0;
    int64_t sched_words = 0;        // int16 words of the packed schedule
    int64_t fac_slots = 0;          // factor values per system (= slots * md)
    int32_t *line_row0 = nullptr;   // [T] first row of each line in solve order
    int32_t *line_len = nullptr;    // [T] rows of each line (0: padding thread)
    int32_t *line_start = nullptr;  // [T] step of each line's first row
    int32_t *bslot = nullptr;       // [nbatch] first slot of each batch
    int32_t *bcount = nullptr;      // [nbatch] slots of each batch (multiple of 8)
    int64_t *boff = nullptr;        // [nbatch] int16 offset of each batch's schedule block
    int16_t *sched = nullptr;       // [sched_words] per batch: header + [slot][md]
    int32_t *vperm = nullptr;       // [fac_slots] factor CSR position (-1 = padding)
};
struct LineSched {
    bool ok = false;
    int32_t nslot = 0;                    // slots per system (multiple of 8)
    std::vector<int32_t> h_rowof, h_slot;  // slot -> row (-1: padding), row -> slot
    int32_t *rowof = nullptr, *slot = nullptr;
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
