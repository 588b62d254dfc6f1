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
// a mesh in natural order). Line l is owned by one lane of one warp; lines
// are rigid: in the forward solve row k of line l is solved at step
// start[l] + k, and the backward solve runs the same steps in reverse.
//
// The schedule qualifies when every cross-line dependency of a row lies on
// the adjacent line (l - 1 forward, l + 1 backward) at most two steps back,
// so a lane's operands are its own previous value (register), and its left
// neighbour's values one and two steps back (one warp shuffle per step; the
// first lane of a warp reads them from a shared-memory ring written by the
// last lane of the previous warp). Every row's dependencies, in the
// reference's summation order, are then a subsequence of the three "kinds"
//     L2 (left line, 2 steps back), L1 (left, 1 step back), S1 (own line),
// and the factor is stored as three values per row (0 where a kind is absent).
//
// Line order ("slots"): lines are placed on lanes 32w + t (forward, padded at
// the front to a multiple of 32); each warp's step range is cut into tiles
// of kTileSteps steps x 32 lanes, element (q / 2) * 64 + 2 t + q % 2 (a
// lane's two steps of a tile half are adjacent: 16-byte loads), and a warp's tiles are
// contiguous, so every pipeline stage of a warp is one bulk copy per array.
// The backward solve traverses the same tiles in reverse (warp W-1-w, lane
// 31-t, element 127-e), so one slot order serves both directions and every
// vector of the PCG loop. Padding slots belong to no row and hold zeros.
constexpr int32_t kTileSteps = 4;
constexpr int32_t kTileSlots = 32 * kTileSteps;
constexpr int32_t kLineKinds = 3;  // L2, L1, S1
// line warps of one CTA (each paired with a helper warp: 16 warps, 512
// threads, <= 128 registers) and CTAs of one system's cluster
constexpr int32_t kLineMaxWarps = 8;
constexpr int32_t kLineMaxClusterCtas = 4;
constexpr int32_t kLineMaxLines = 32 * kLineMaxWarps * kLineMaxClusterCtas;  // 1024

struct LineDir {
    int32_t warps = 0;
    int32_t ntiles = 0;              // tiles in all (nslot / kTileSlots)
    int32_t max_warp_tiles = 0;      // most tiles of one warp
    int32_t ring = 64;               // steps per warp's outgoing value ring (power of two)
    int64_t fac_slots = 0;           // factor values per system (= nslot * kLineKinds)
    std::vector<int32_t> h_meta;     // [warps][4]: first step, tiles, first tile, 0
    int32_t *meta = nullptr;         // device copy of h_meta
    int32_t *vperm = nullptr;        // [tile][kind][element]: CSR position of the factor value (-1 = zero)
};
struct LineSched {
    bool ok = false;
    int32_t nslot = 0;                     // slots per system (multiple of kTileSlots)
    int32_t lines = 0, steps = 0;
    std::vector<int32_t> h_rowof, h_slot;  // slot -> row (-1: padding), row -> slot
    int32_t *rowof = nullptr, *slot = nullptr;
    LineDir fwd, bwd;
    ~LineSched();
};

// Global level sets of the two triangular solves (trsv_level.cu): rows in
// level order, each row's dependencies in the reference's summation order
// (sparse.py:222-239: ascending columns forward, the column scatter's
// descending order backward). The level-synchronous kernel walks the levels
// with one grid-wide barrier each; used for patterns without a line
// schedule (3-D meshes) when the batch gives every level enough work.
struct LevelDir {
    int32_t nlev = 0, max_rows = 0;
    int64_t entries = 0;
    int32_t *lvl_ptr = nullptr;  // [nlev + 1] into rows
    int32_t *rows = nullptr;     // [n] rows in level order
    int32_t *eptr = nullptr;     // [n + 1] dependency range of the k-th row in level order
    int32_t *ecol = nullptr;     // [entries] dependency row
    int32_t *sperm = nullptr;    // [entries] CSR position of the factor value
};
struct LevelSched {
    LevelDir fwd, bwd;
    ~LevelSched();
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
    std::unique_ptr<LevelSched> levels;                    // built on first use
    std::mutex mu;
    ~Pattern();
    // Schedule for `chunk_rows` (built on first use); nullptr + err on failure.
    SchedSet *schedule(int32_t chunk_rows, std::string &err);
    // Line schedule, or nullptr when the pattern does not qualify.
    LineSched *line_schedule();
    // Global level sets (nullptr without a factor analysis or on allocation failure).
    LevelSched *level_schedule();
};

// Rows per chunk for a solve over B columns in groups of G (heuristic,
// overridable with NPCG_CHUNK_ROWS).
int32_t choose_chunk_rows(int64_t n, int B, int G);

}  // namespace npcg
