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
#include <climits>
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
    int32_t **ptrs[] = {&s.packed, &s.lvl_woff, &s.lvl_meta, &s.chunk_lvl, &s.sperm};
    for (auto p : ptrs) {
        if (*p) cudaFree(*p);
        *p = nullptr;
    }
}

SchedSet::~SchedSet() {
    free_schedule(fwd);
    free_schedule(bwd);
}

Pattern::~Pattern() {
    scheds.clear();
    int32_t **ptrs[] = {&rp, &col, &dp, &pair, &lower_slot, &src};
    for (auto p : ptrs)
        if (*p) cudaFree(*p);
}

// Build one direction. `upper` selects the backward (transpose) solve: rows
// are visited in descending order, depend on their upper entries, and each
// row's entries are accumulated in descending column order -- the order in
// which the reference's column scatter (sparse.py:236-239) subtracts them.
// Chunk boundaries near multiples of R, preferring rows that do not depend on
// their predecessor (row i-1 absent from row i's lower pattern). On meshes in
// natural order those are the starts of grid lines; cutting there keeps the
// chunk-local level structure aligned with the global one (window ~3 levels).
// A cut inside a line would make the next chunk's first levels wait on the
// previous chunk's last ones and serialise the chunks.
static std::vector<int32_t> chunk_bounds(const Pattern &P, int32_t R) {
    const int32_t n = (int32_t)P.n;
    std::vector<int32_t> cand;
    for (int32_t i = 1; i < n; ++i) {
        bool dep_prev = false;
        for (int32_t p = P.h_rp[i]; p < P.h_dp[i]; ++p) dep_prev |= P.h_col[p] == i - 1;
        if (!dep_prev) cand.push_back(i);
    }
    std::vector<int32_t> b{0};
    while (b.back() < n) {
        const int64_t target = (int64_t)b.back() + R;
        if (target >= n) break;
        int32_t cut = (int32_t)target;
        auto it = std::lower_bound(cand.begin(), cand.end(), (int32_t)target);
        int64_t best = -1;
        if (it != cand.end()) best = *it;
        if (it != cand.begin() && *(it - 1) > b.back()) {
            const int32_t lo = *(it - 1);
            if (best < 0 || target - lo <= best - target) best = lo;
        }
        if (best > b.back() && std::llabs(best - target) <= R / 2) cut = (int32_t)best;
        b.push_back(cut);
    }
    b.push_back(n);
    return b;
}

static std::string build_direction(const Pattern &P, int32_t R, bool upper, Schedule &S) {
    const int32_t n = (int32_t)P.n;
    const auto &rp = P.h_rp, &col = P.h_col, &dp = P.h_dp;
    const std::vector<int32_t> bounds = n ? chunk_bounds(P, R) : std::vector<int32_t>{0};
    const int32_t C = (int32_t)bounds.size() - 1;
    std::vector<int32_t> cid(n);
    for (int32_t c = 0; c < C; ++c)
        for (int32_t i = bounds[c]; i < bounds[c + 1]; ++i) cid[i] = upper ? C - 1 - c : c;
    auto chunk_of = [&](int32_t i) { return cid[i]; };
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

    std::vector<int32_t> chunk_lvl(C + 1, 0), nlev(C, 0);
    for (int32_t i = 0; i < n; ++i) nlev[chunk_of(i)] = std::max(nlev[chunk_of(i)], lvl[i] + 1);
    for (int32_t c = 0; c < C; ++c) chunk_lvl[c + 1] = chunk_lvl[c] + nlev[c];
    const int32_t TL = chunk_lvl[C];
    std::vector<int32_t> lvl_ptr(TL + 1, 0);
    for (int32_t i = 0; i < n; ++i) lvl_ptr[chunk_lvl[chunk_of(i)] + lvl[i] + 1]++;
    int32_t maxw = 1, max_chunk_levels = 0;
    for (int32_t L = 0; L < TL; ++L) {
        maxw = std::max(maxw, lvl_ptr[L + 1]);
        lvl_ptr[L + 1] += lvl_ptr[L];
    }
    for (int32_t c = 0; c < C; ++c) max_chunk_levels = std::max(max_chunk_levels, nlev[c]);
    // rows in (chunk, level, visit order): stable counting sort
    std::vector<int32_t> rows(n), fill(lvl_ptr.begin(), lvl_ptr.end() - 1), pos(n);
    for (int32_t t = 0; t < n; ++t) {
        const int32_t i = upper ? n - 1 - t : t;
        const int32_t L = chunk_lvl[chunk_of(i)] + lvl[i];
        pos[i] = fill[L] - lvl_ptr[L];
        rows[fill[L]++] = i;
    }
    // Packed per-level blocks (int32 words, every section padded to 16 B so a
    // level is one TMA bulk copy):
    //   rows[nrow] | eoff[nrow+1] (entry offsets within the level) |
    //   dep[ne] (>=0 ring slot, <0: -(x+1) = index into xrow) | xrow[nx]
    // Factor values live in a separate array in the same level order, each
    // level padded to an even entry count (sperm maps it back to CSR).
    auto pad4 = [](int64_t x) { return (x + 3) & ~int64_t(3); };
    std::vector<int32_t> packed, lvl_woff(TL + 1, 0), meta(4 * (size_t)TL, 0), sperm;
    int32_t max_words = 0, max_se = 0, maxx = 0;
    int64_t entries = 0;
    for (int32_t L = 0; L < TL; ++L) {
        const int32_t s0 = lvl_ptr[L], s1 = lvl_ptr[L + 1], nrow = s1 - s0;
        std::vector<int32_t> eoff{0}, dep, xrow, perm;
        for (int32_t s = s0; s < s1; ++s) {
            const int32_t i = rows[s];
            const int32_t ci = chunk_of(i);
            auto push = [&](int32_t p) {
                const int32_t j = col[p];
                if (chunk_of(j) == ci) {
                    dep.push_back((lvl[j] % window) * maxw + pos[j]);
                } else {
                    xrow.push_back(j);
                    dep.push_back(-(int32_t)xrow.size());
                }
                perm.push_back(p);
            };
            if (upper)
                for (int32_t p = dep_end(i) - 1; p >= dep_begin(i); --p) push(p);
            else
                for (int32_t p = dep_begin(i); p < dep_end(i); ++p) push(p);
            eoff.push_back((int32_t)dep.size());
        }
        const int32_t ne = (int32_t)dep.size(), nx = (int32_t)xrow.size();
        const int64_t w0 = (int64_t)packed.size();
        auto put = [&](const std::vector<int32_t> &v, int64_t len) {
            packed.insert(packed.end(), v.begin(), v.end());
            packed.resize(packed.size() + (pad4(len) - len), 0);
        };
        put(std::vector<int32_t>(rows.begin() + s0, rows.begin() + s1), nrow);
        put(eoff, nrow + 1);
        put(dep, ne);
        put(xrow, nx);
        lvl_woff[L + 1] = (int32_t)packed.size();
        max_words = std::max<int32_t>(max_words, (int32_t)(packed.size() - w0));
        const int32_t se = (ne + 1) & ~1;
        meta[4 * L + 0] = nrow;
        meta[4 * L + 1] = ne;
        meta[4 * L + 2] = nx;
        meta[4 * L + 3] = (int32_t)sperm.size();
        sperm.insert(sperm.end(), perm.begin(), perm.end());
        sperm.resize(sperm.size() + (se - ne), -1);
        max_se = std::max(max_se, se);
        maxx = std::max(maxx, nx);
        entries += ne;
    }
    free_schedule(S);
    S.chunks = C;
    S.chunk_rows = R;
    S.window = window;
    S.maxw = maxw;
    S.total_levels = TL;
    S.max_chunk_levels = max_chunk_levels;
    S.levels_global = levels_global;
    S.entries = entries;
    S.padded_entries = (int64_t)sperm.size();
    S.max_words = max_words;
    S.max_se = max_se;
    S.maxx = maxx;
    S.packed = upload(packed);
    S.lvl_woff = upload(lvl_woff);
    S.lvl_meta = upload(meta);
    S.chunk_lvl = upload(chunk_lvl);
    S.sperm = upload(sperm);
    if (!S.packed || !S.lvl_woff || !S.lvl_meta || !S.chunk_lvl || !S.sperm)
        return "cudaMalloc failed for the solve schedule";
    return "";
}

LineSched::~LineSched() {
    if (rowof) cudaFree(rowof);
    if (slot) cudaFree(slot);
    for (LineDir *d : {&fwd, &bwd}) {
        if (d->meta) cudaFree(d->meta);
        if (d->vperm) cudaFree(d->vperm);
    }
}

// The line schedule of a structurally symmetric pattern (pattern.h); false
// when it does not qualify (too many lines, a dependency off the adjacent
// line or more than two steps back, an order the three kinds cannot carry).
//
// Forward: rows of line l run at steps start[l] + k, start[l] the earliest
// step at which every cross-line dependency of the line is solved at least a
// step earlier. Backward runs the steps in reverse: an upper dependency c of
// row i has row i as a lower dependency, so it was solved at a later forward
// step -- an earlier backward one -- at the same distance.
static bool build_line_sched(const Pattern &P, LineSched &LS) {
    const int32_t n = (int32_t)P.n;
    const auto &rp = P.h_rp, &col = P.h_col, &dp = P.h_dp;
    if (n == 0) return false;
    std::vector<int32_t> starts{0};
    for (int32_t i = 1; i < n; ++i) {
        bool dep_prev = false;
        for (int32_t p = rp[i]; p < dp[i]; ++p) dep_prev |= col[p] == i - 1;
        if (!dep_prev) starts.push_back(i);
    }
    starts.push_back(n);
    const int32_t L = (int32_t)starts.size() - 1;
    if (L > kLineMaxLines) return false;
    std::vector<int32_t> line(n), pos(n), lstart(L, 0);
    for (int32_t l = 0; l < L; ++l)
        for (int32_t i = starts[l]; i < starts[l + 1]; ++i) {
            line[i] = l;
            pos[i] = i - starts[l];
        }
    int32_t steps = 0;
    for (int32_t l = 0; l < L; ++l) {
        int32_t st = 0;
        for (int32_t i = starts[l]; i < starts[l + 1]; ++i)
            for (int32_t p = rp[i]; p < dp[i]; ++p) {
                const int32_t j = col[p];
                if (line[j] != l) st = std::max(st, lstart[line[j]] + pos[j] + 1 - pos[i]);
            }
        lstart[l] = st;
        steps = std::max(steps, st + starts[l + 1] - starts[l]);
    }
    auto fstep = [&](int32_t i) { return lstart[line[i]] + pos[i]; };
    // kind of the dependency of row i on row j (0 = L2, 1 = L1, 2 = S1), -1 if none fits
    auto kind = [&](int32_t i, int32_t j, bool upper) -> int32_t {
        const int32_t li = line[i], lj = line[j];
        if (lj == li) return j == i + (upper ? 1 : -1) ? 2 : -1;
        if (lj != li + (upper ? 1 : -1)) return -1;
        const int32_t age = upper ? fstep(j) - fstep(i) : fstep(i) - fstep(j);
        return age == 1 ? 1 : (age == 2 ? 0 : -1);
    };
    // every row's dependencies, in the reference's order (sparse.py:222-239:
    // ascending columns forward, the column scatter's descending order
    // backward), must be strictly increasing kinds
    std::vector<int32_t> kpos_f((size_t)n * kLineKinds, -1), kpos_b((size_t)n * kLineKinds, -1);
    for (int32_t i = 0; i < n; ++i) {
        int32_t last = -1;
        for (int32_t p = rp[i]; p < dp[i]; ++p) {
            const int32_t k = kind(i, col[p], false);
            if (k <= last) return false;
            kpos_f[(size_t)i * kLineKinds + k] = p;
            last = k;
        }
        last = -1;
        for (int32_t p = rp[i + 1] - 1; p > dp[i]; --p) {
            const int32_t k = kind(i, col[p], true);
            if (k <= last) return false;
            kpos_b[(size_t)i * kLineKinds + k] = p;
            last = k;
        }
    }
    const int32_t W = (L + 31) / 32, pad = 32 * W - L;
    // forward tiles of every warp
    std::vector<int32_t> s0(W, INT32_MAX), s1(W, 0), nt(W), t0(W);
    for (int32_t l = 0; l < L; ++l) {
        const int32_t w = (l + pad) / 32;
        s0[w] = std::min(s0[w], lstart[l]);
        s1[w] = std::max(s1[w], lstart[l] + starts[l + 1] - starts[l]);
    }
    int32_t tiles = 0, maxt = 0;
    for (int32_t w = 0; w < W; ++w) {
        nt[w] = (s1[w] - s0[w] + kTileSteps - 1) / kTileSteps;
        t0[w] = tiles;
        tiles += nt[w];
        maxt = std::max(maxt, nt[w]);
    }
    if ((int64_t)tiles * kTileSlots > INT32_MAX / kLineKinds) return false;
    const int32_t nslot = tiles * kTileSlots;
    LS.nslot = nslot;
    LS.lines = L;
    LS.steps = steps;
    LS.h_rowof.assign(nslot, -1);
    LS.h_slot.assign(n, -1);
    for (int32_t i = 0; i < n; ++i) {
        const int32_t q = line[i] + pad, w = q / 32, d = fstep(i) - s0[w];
        const int32_t qs = d % kTileSteps;  // a lane's steps 2h, 2h+1 are adjacent
        const int32_t slot = (t0[w] + d / kTileSteps) * kTileSlots + (qs >> 1) * 64 + (q % 32) * 2 + (qs & 1);
        LS.h_slot[i] = slot;
        LS.h_rowof[slot] = i;
    }
    auto build_dir = [&](bool upper, LineDir &D) -> bool {
        D.warps = W;
        D.ntiles = tiles;
        D.max_warp_tiles = maxt;
        D.fac_slots = (int64_t)nslot * kLineKinds;
        int32_t lag = 0;  // largest first-step offset between adjacent warps
        for (int32_t w = 0; w + 1 < W; ++w) lag = std::max(lag, std::abs(s0[w + 1] - s0[w]));
        D.ring = 64;
        while (D.ring < 2 * lag + 16) D.ring *= 2;
        D.h_meta.assign((size_t)W * 4, 0);
        for (int32_t wd = 0; wd < W; ++wd) {
            const int32_t w = upper ? W - 1 - wd : wd;  // forward warp
            int32_t *m = &D.h_meta[(size_t)wd * 4];
            m[0] = upper ? steps - s0[w] - kTileSteps * nt[w] : s0[w];
            m[1] = nt[w];
            m[2] = t0[w];
        }
        std::vector<int32_t> vperm((size_t)D.fac_slots, -1);
        const auto &kp = upper ? kpos_b : kpos_f;
        for (int32_t slot = 0; slot < nslot; ++slot) {
            const int32_t i = LS.h_rowof[slot];
            if (i < 0) continue;
            const int32_t tile = slot / kTileSlots, e = slot % kTileSlots;
            const int32_t ed = upper ? kTileSlots - 1 - e : e;  // element in this direction's traversal
            for (int32_t k = 0; k < kLineKinds; ++k)
                vperm[((size_t)tile * kLineKinds + k) * kTileSlots + ed] = kp[(size_t)i * kLineKinds + k];
        }
        D.meta = upload(D.h_meta);
        D.vperm = upload(vperm);
        return D.meta && D.vperm;
    };
    if (!build_dir(false, LS.fwd) || !build_dir(true, LS.bwd)) return false;
    LS.rowof = upload(LS.h_rowof);
    LS.slot = upload(LS.h_slot);
    return LS.rowof && LS.slot;
}

LevelSched::~LevelSched() {
    for (LevelDir *d : {&fwd, &bwd})
        for (int32_t *p : {d->lvl_ptr, d->rows, d->eptr, d->ecol, d->sperm})
            if (p) cudaFree(p);
}

static bool build_level_dir(const Pattern &P, bool upper, LevelDir &D) {
    const int32_t n = (int32_t)P.n;
    const auto &rp = P.h_rp, &col = P.h_col, &dp = P.h_dp;
    std::vector<int32_t> lvl(n, 0);
    int32_t nlev = n ? 1 : 0;
    for (int32_t t = 0; t < n; ++t) {  // processing order: ascending rows forward, descending backward
        const int32_t i = upper ? n - 1 - t : t;
        int32_t l = 0;
        const int32_t p0 = upper ? dp[i] + 1 : rp[i], p1 = upper ? rp[i + 1] : dp[i];
        for (int32_t p = p0; p < p1; ++p) l = std::max(l, lvl[col[p]] + 1);
        lvl[i] = l;
        nlev = std::max(nlev, l + 1);
    }
    std::vector<int32_t> lvl_ptr(nlev + 1, 0);
    for (int32_t i = 0; i < n; ++i) lvl_ptr[lvl[i] + 1]++;
    int32_t max_rows = 0;
    for (int32_t L = 0; L < nlev; ++L) {
        max_rows = std::max(max_rows, lvl_ptr[L + 1]);
        lvl_ptr[L + 1] += lvl_ptr[L];
    }
    std::vector<int32_t> rows(n), fill(lvl_ptr.begin(), lvl_ptr.end() - 1);
    for (int32_t t = 0; t < n; ++t) {
        const int32_t i = upper ? n - 1 - t : t;
        rows[fill[lvl[i]]++] = i;
    }
    std::vector<int32_t> eptr(n + 1, 0), ecol, sperm;
    for (int32_t k = 0; k < n; ++k) {
        const int32_t i = rows[k];
        if (upper)  // the column scatter's order: descending columns (sparse.py:236-239)
            for (int32_t p = rp[i + 1] - 1; p > dp[i]; --p) ecol.push_back(col[p]), sperm.push_back(p);
        else
            for (int32_t p = rp[i]; p < dp[i]; ++p) ecol.push_back(col[p]), sperm.push_back(p);
        eptr[k + 1] = (int32_t)ecol.size();
    }
    D.nlev = nlev;
    D.max_rows = max_rows;
    D.entries = (int64_t)ecol.size();
    D.lvl_ptr = upload(lvl_ptr);
    D.rows = upload(rows);
    D.eptr = upload(eptr);
    D.ecol = upload(ecol);
    D.sperm = upload(sperm);
    return D.lvl_ptr && D.rows && D.eptr && D.ecol && D.sperm;
}

LevelSched *Pattern::level_schedule() {
    std::lock_guard<std::mutex> lock(mu);
    if (!factor_ok) return nullptr;
    if (!levels) {
        auto L = std::make_unique<LevelSched>();
        if (!build_level_dir(*this, false, L->fwd) || !build_level_dir(*this, true, L->bwd)) return nullptr;
        levels = std::move(L);
    }
    return levels.get();
}

LineSched *Pattern::line_schedule() {
    std::lock_guard<std::mutex> lock(mu);
    if (!factor_ok) return nullptr;
    if (!lines) {
        lines = std::make_unique<LineSched>();
        lines->ok = !std::getenv("NPCG_NO_LINES") && build_line_sched(*this, *lines);
    }
    return lines->ok ? lines.get() : nullptr;
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
    err = build_direction(*this, R, false, set->fwd);
    if (err.empty()) err = build_direction(*this, R, true, set->bwd);
    if (!err.empty()) return nullptr;
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
    // The solve is latency bound along the level chain; extra chunks only add
    // hand-offs. Use just enough chunks for ~2 resident units per SM, each of
    // at least 4096 rows.
    int64_t chunks = (2 * 148 + groups - 1) / groups;
    chunks = std::max<int64_t>(1, std::min<int64_t>(chunks, n / 4096));
    return (int32_t)((n + chunks - 1) / chunks);
}

}  // namespace npcg
