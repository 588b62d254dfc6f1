// pattern.h -- device-resident analysis of one sparsity pattern (internal).
#pragma once
#include <cstdint>
#include <string>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

namespace npcg {

// One direction (forward = lower rows ascending, backward = upper rows
// descending) of the chunked triangular-solve schedule. Rows are split into
// contiguous chunks; inside a chunk rows are grouped by chunk-local level
// (longest intra-chunk dependency chain). A CTA owning a (chunk, batch
// group) unit walks its levels with one __syncthreads per level, keeping
// the freshly solved values in a shared-memory ring of `window` levels.
// Dependencies on earlier chunks are satisfied by per-(chunk, group)
// progress counters published with release stores.
struct Schedule {
    int32_t chunks = 0;       // number of chunks (processing order)
    int32_t chunk_rows = 0;   // rows per chunk (last may be short)
    int32_t window = 1;       // ring depth in levels
    int32_t maxw = 1;         // max rows in one chunk-local level
    int32_t total_levels = 0; // sum over chunks of their level counts
    int32_t max_chunk_levels = 0;
    int32_t levels_global = 0;
    bool smem_ok = true;      // ring fits; else all deps read from global
    // device arrays
    int32_t *rows = nullptr;      // [n] row ids in (chunk, level, position) order
    int32_t *lvl_ptr = nullptr;   // [total_levels+1] offsets into rows
    int32_t *chunk_lvl = nullptr; // [chunks+1] offsets into lvl_ptr
    int32_t *req_ptr = nullptr;   // [total_levels+1] offsets into req_*
    int32_t *req_chunk = nullptr; // external requirement: chunk (processing index)
    int32_t *req_lvl = nullptr;   //   ... must have completed this local level
    int32_t *row_slot = nullptr;  // [n] ring slot of each row (level%W*maxw+pos)
};

// Both directions for one chunk size, plus the per-entry operand array:
// dep[p] >= 0 is a ring slot (same chunk), dep[p] < 0 encodes row -(dep+1).
// Lower entries carry forward operands, upper entries backward operands.
struct SchedSet {
    Schedule fwd, bwd;
    int32_t *dep = nullptr;
    ~SchedSet();
};

struct Pattern {
    int64_t n = 0, nnz = 0, nnz_lower = 0;
    bool full_diag = false, symmetric = false, factor_ok = false;
    std::vector<int32_t> h_rp, h_col, h_dp, h_pair;
    int32_t *rp = nullptr, *col = nullptr, *dp = nullptr, *pair = nullptr;
    int32_t *lower_slot = nullptr; // [nnz_lower] CSR position of each strict-lower entry
    int32_t *src = nullptr;        // [nnz] row of each stored entry (edge source, gnn.py:83)
    std::map<int32_t, std::unique_ptr<SchedSet>> scheds;  // by chunk rows
    std::mutex mu;
    ~Pattern();
    // Schedule for `chunk_rows` (built on first use); nullptr + err on failure.
    SchedSet *schedule(int32_t chunk_rows, std::string &err);
};

// Rows per chunk for a solve over B columns in groups of G (heuristic,
// overridable with NPCG_CHUNK_ROWS).
int32_t choose_chunk_rows(int64_t n, int B, int G);

}  // namespace npcg
