// pattern.cpp -- one-time host analysis of a sparsity pattern.
//
// Replaces, once per mesh, the pattern work the reference redoes on every
// call: CSR validation (pkg/src/pcgkit/sparse.py:44-65), full-diagonal and
// symmetry checks (sparse.py:133-147), the reverse-edge index of
// graph_from_system (gnn.py:83-88), the strict-lower slot order of
// A.strict_lower() (sparse.py:149-153, gnn.py:278-281) and -- new on the
// GPU -- the dependency schedules of the two triangular solves that
// ldlt_apply_inverse runs sequentially (sparse.py:222-239).
#include "pattern.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

namespace npcg {

template <class T>
static T *upload(const std::vector<T> &v) {
    T *d = nullptr;
    size_t bytes = std::max<size_t>(1, v.size()) * sizeof(T);
    if (cudaMalloc(&d, bytes) != cudaSuccess) return nullptr;
    if (!v.empty() && cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaFree(d);
        return nullptr;
    }
    return d;
}

static void free_schedule(Schedule &s) {
    int32_t **ptrs[] = {&s.rows, &s.lvl_ptr, &s.chunk_lvl, &s.req_ptr,
                        &s.req_chunk, &s.req_lvl, &s.row_slot};
    for (auto p : ptrs) {
        if (*p) cudaFree(*p);
        *p = nullptr;
    }
}

SchedSet::~SchedSet() {
    free_schedule(fwd);
    free_schedule(bwd);
    if (dep) cudaFree(dep);
}

Pattern::~Pattern() {
    scheds.clear();
    int32_t **ptrs[] = {&rp, &col, &dp, &pair, &lower_slot, &src};
    for (auto p : ptrs)
        if (*p) cudaFree(*p);
}

// Build one direction. `upper` selects the backward (transpose) solve:
// rows are visited in descending order and depend on their upper entries.
static std::string build_direction(const Pattern &P, int32_t R, bool upper,
                                   Schedule &S, std::vector<int32_t> &dep_h) {
    const int32_t n = (int32_t)P.n;
    const auto &rp = P.h_rp, &col = P.h_col, &dp = P.h_dp;
    const int32_t C = n == 0 ? 0 : (n + R - 1) / R;
    // processing index of the chunk holding row i
    auto chunk_of = [&](int32_t i) { return upper ? (C - 1 - i / R) : i / R; };
    auto dep_begin = [&](int32_t i) { return upper ? dp[i] + 1 : rp[i]; };
    auto dep_end = [&](int32_t i) { return upper ? rp[i + 1] : dp[i]; };

    std::vector<int32_t> lvl(n, 0), glev(n, 0);
    int32_t window = 1, levels_global = 0;
    for (int32_t t = 0; t < n; ++t) {
        const int32_t i = upper ? n - 1 - t : t;
        const int32_t ci = chunk_of(i);
        int32_t l = 0, g = 0;
        for (int32_t p = dep_begin(i); p < dep_end(i); ++p) {
            const int32_t j = col[p];
            g = std::max(g, glev[j] + 1);
            if (chunk_of(j) == ci) l = std::max(l, lvl[j] + 1);
        }
        lvl[i] = l;
        glev[i] = g;
        levels_global = std::max(levels_global, g + 1);
    }
    for (int32_t i = 0; i < n; ++i)
        for (int32_t p = dep_begin(i); p < dep_end(i); ++p) {
            const int32_t j = col[p];
            if (chunk_of(j) == chunk_of(i)) window = std::max(window, lvl[i] - lvl[j] + 1);
        }

    // per chunk: level counts -> offsets
    std::vector<int32_t> chunk_lvl(C + 1, 0);
    std::vector<int32_t> nlev(C, 0);
    for (int32_t i = 0; i < n; ++i) nlev[chunk_of(i)] = std::max(nlev[chunk_of(i)], lvl[i] + 1);
    for (int32_t c = 0; c < C; ++c) chunk_lvl[c + 1] = chunk_lvl[c] + nlev[c];
    const int32_t TL = chunk_lvl[C];
    std::vector<int32_t> lvl_cnt(TL + 1, 0);
    for (int32_t i = 0; i < n; ++i) lvl_cnt[chunk_lvl[chunk_of(i)] + lvl[i] + 1]++;
    std::vector<int32_t> lvl_ptr(TL + 1, 0);
    int32_t maxw = 1, max_chunk_levels = 0;
    for (int32_t L = 0; L < TL; ++L) {
        lvl_ptr[L + 1] = lvl_ptr[L] + lvl_cnt[L + 1];
        maxw = std::max(maxw, lvl_cnt[L + 1]);
    }
    for (int32_t c = 0; c < C; ++c) max_chunk_levels = std::max(max_chunk_levels, nlev[c]);
    // rows in (chunk, level, row-visit order): stable counting sort
    std::vector<int32_t> rows(n), fill(lvl_ptr.begin(), lvl_ptr.end() - 1), pos(n), slot(n);
    for (int32_t t = 0; t < n; ++t) {
        const int32_t i = upper ? n - 1 - t : t;
        const int32_t L = chunk_lvl[chunk_of(i)] + lvl[i];
        pos[i] = fill[L] - lvl_ptr[L];
        rows[fill[L]++] = i;
    }
    for (int32_t i = 0; i < n; ++i) slot[i] = (lvl[i] % window) * maxw + pos[i];
    // dependency operands and external requirements
    std::vector<int32_t> req_ptr(TL + 1, 0), req_chunk, req_lvl;
    std::vector<int32_t> best;  // scratch: per level, max needed level per chunk
    for (int32_t c = 0; c < C; ++c) {
        for (int32_t l = 0; l < nlev[c]; ++l) {
            const int32_t L = chunk_lvl[c] + l;
            std::vector<std::pair<int32_t, int32_t>> need;  // (chunk, level)
            for (int32_t s = lvl_ptr[L]; s < lvl_ptr[L + 1]; ++s) {
                const int32_t i = rows[s];
                for (int32_t p = dep_begin(i); p < dep_end(i); ++p) {
                    const int32_t j = col[p];
                    const int32_t cj = chunk_of(j);
                    if (cj == c) {
                        dep_h[p] = slot[j];
                    } else {
                        dep_h[p] = -(j + 1);
                        need.emplace_back(cj, lvl[j]);
                    }
                }
            }
            std::sort(need.begin(), need.end());
            for (size_t k = 0; k < need.size(); ++k) {
                if (k + 1 < need.size() && need[k + 1].first == need[k].first) continue;
                req_chunk.push_back(need[k].first);
                req_lvl.push_back(need[k].second);
            }
            req_ptr[L + 1] = (int32_t)req_chunk.size();
        }
    }
    free_schedule(S);
    S.chunks = C;
    S.chunk_rows = R;
    S.window = window;
    S.maxw = maxw;
    S.total_levels = TL;
    S.max_chunk_levels = max_chunk_levels;
    S.levels_global = levels_global;
    S.rows = upload(rows);
    S.lvl_ptr = upload(lvl_ptr);
    S.chunk_lvl = upload(chunk_lvl);
    S.req_ptr = upload(req_ptr);
    S.req_chunk = upload(req_chunk);
    S.req_lvl = upload(req_lvl);
    S.row_slot = upload(slot);
    if (!S.rows || !S.lvl_ptr || !S.chunk_lvl || !S.req_ptr || !S.req_chunk || !S.req_lvl || !S.row_slot)
        return "cudaMalloc failed for the solve schedule";
    return "";
}

SchedSet *Pattern::schedule(int32_t R, std::string &err) {
    std::lock_guard<std::mutex> lock(mu);
    if (!factor_ok) {
        err = "pattern has no factor analysis (needs a full diagonal and symmetric structure)";
        return nullptr;
    }
    if (R < 1) R = 1;
    if (n > 0 && R > n) R = (int32_t)n;
    auto it = scheds.find(R);
    if (it != scheds.end()) return it->second.get();
    auto set = std::make_unique<SchedSet>();
    std::vector<int32_t> dep_h(nnz, 0);
    err = build_direction(*this, R, false, set->fwd, dep_h);
    if (err.empty()) err = build_direction(*this, R, true, set->bwd, dep_h);
    if (!err.empty()) return nullptr;
    set->dep = upload(dep_h);
    if (!set->dep) {
        err = "cudaMalloc failed for the dependency operands";
        return nullptr;
    }
    SchedSet *raw = set.get();
    scheds.emplace(R, std::move(set));
    return raw;
}

int32_t choose_chunk_rows(int64_t n, int B, int G) {
    if (const char *env = std::getenv("NPCG_CHUNK_ROWS")) {
        const long v = std::atol(env);
        if (v > 0) return (int32_t)std::min<int64_t>(v, std::max<int64_t>(n, 1));
    }
    if (n <= 0) return 1;
    const int groups = (B + G - 1) / G;
    // aim for ~3 resident units per SM across all groups, chunks of >= 256 rows
    int64_t chunks = (3 * 148 + groups - 1) / groups;
    chunks = std::max<int64_t>(1, std::min<int64_t>(chunks, n / 256));
    return (int32_t)((n + chunks - 1) / chunks);
}

}  // namespace npcg
