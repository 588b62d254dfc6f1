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
        void *ptrs[] = {d->line_row0, d->line_len, d->line_start, d->bslot, d->bcount, d->boff, d->sched, d->vperm};
        for (void *q : ptrs)
            if (q) cudaFree(q);
    }
}

// The line schedule of a structurally symmetric pattern; false when it does
// not qualify (too many lines, deep cross-line window, wide rows).
//
// Forward: rows of line l run at steps start[l] + k, start[l] the earliest
// step at which every cross-line dependency of the line is solved a step
// earlier (a row's dependencies lie in earlier lines or earlier in its own
// line). Backward runs the padded step range in reverse: an upper
// dependency j of row i has row i as a lower dependency, so it was solved
// at a later forward step -- an earlier backward one -- and the ring window
// that covers the forward distances covers the backward ones.
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
    int32_t steps = 0, md = 1;
    for (int32_t l = 0; l < L; ++l) {
        int32_t st = 0;
        for (int32_t i = starts[l]; i < starts[l + 1]; ++i) {
            md = std::max(md, std::max(dp[i] - rp[i], rp[i + 1] - dp[i] - 1));
            for (int32_t p = rp[i]; p < dp[i]; ++p) {
                const int32_t j = col[p];
                if (line[j] != l) st = std::max(st, lstart[line[j]] + pos[j] + 1 - pos[i]);
            }
        }
        lstart[l] = st;
        steps = std::max(steps, st + starts[l + 1] - starts[l]);
    }
    auto fstep = [&](int32_t i) { return lstart[line[i]] + pos[i]; };
    int32_t span = 1;
    for (int32_t i = 0; i < n; ++i)
        for (int32_t p = rp[i]; p < dp[i]; ++p) {
            const int32_t j = col[p];
            if (j == i - 1 && line[j] == line[i]) continue;  // carried in a register
            span = std::max(span, fstep(i) - fstep(j) + 1);
        }
    int32_t W = 1;
    while (W < span) W <<= 1;
    if (W > 16 || md > 8) return false;
    const int32_t MD = md <= 2 ? 2 : (md <= 3 ? 3 : (md <= 4 ? 4 : 8));
    const int32_t T = (L + 31) & ~31;
    const int32_t K = kLineBatch;
    const int32_t SP = (steps + K - 1) / K * K, nb = SP / K;
    // active line range of every step -> slots
    std::vector<int32_t> lo(SP, INT32_MAX), hi(SP, 0), off(SP, 0);
    for (int32_t l = 0; l < L; ++l)
        for (int32_t s = lstart[l]; s < lstart[l] + starts[l + 1] - starts[l]; ++s) {
            lo[s] = std::min(lo[s], l);
            hi[s] = std::max(hi[s], l + 1);
        }
    std::vector<int32_t> bslot(nb), bcount(nb);
    int32_t cur = 0;
    for (int32_t j = 0; j < nb; ++j) {
        bslot[j] = cur;
        for (int32_t q = 0; q < K; ++q) {
            const int32_t s = j * K + q;
            if (hi[s] == 0) lo[s] = hi[s] = 0;
            off[s] = cur;
            cur += hi[s] - lo[s];
        }
        cur = (cur + kLineSlotAlign - 1) / kLineSlotAlign * kLineSlotAlign;
        bcount[j] = cur - bslot[j];
    }
    const int32_t nslot = cur;
    if ((int64_t)nslot > (int64_t)4 * n + 64 * nb) return false;  // far too sparse a wavefront
    LS.nslot = nslot;
    LS.h_rowof.assign(nslot, -1);
    LS.h_slot.assign(n, -1);
    for (int32_t i = 0; i < n; ++i) {
        const int32_t s = fstep(i);
        const int32_t q = off[s] + line[i] - lo[s];
        LS.h_slot[i] = q;
        LS.h_rowof[q] = i;
    }
    const int32_t zslot = W * T;
    auto build_dir = [&](bool upper, LineDir &D) -> bool {
        std::vector<int32_t> row0(T, 0), llen(T, 0), lst(T, 0), db(nb), dc(nb);
        for (int32_t l = 0; l < L; ++l) {
            const int32_t len = starts[l + 1] - starts[l];
            row0[l] = upper ? starts[l + 1] - 1 : starts[l];
            llen[l] = len;
            lst[l] = upper ? SP - lstart[l] - len : lstart[l];
        }
        std::vector<int64_t> boff(nb);
        std::vector<int16_t> sched;
        std::vector<int32_t> vperm;
        int32_t maxs = 0;
        for (int32_t jd = 0; jd < nb; ++jd) {
            const int32_t j = upper ? nb - 1 - jd : jd;  // forward batch
            db[jd] = bslot[j];
            dc[jd] = bcount[j];
            maxs = std::max(maxs, bcount[j]);
            boff[jd] = (int64_t)sched.size();
            for (int32_t q = 0; q < kLineHeader; ++q) {  // header: int32 base per step, as int16 pairs
                const int32_t s = upper ? j * K + (K - 1 - q) : j * K + q;
                const int32_t base = q < K ? off[s] - lo[s] - bslot[j] : 0;
                sched.push_back((int16_t)(base & 0xffff));
                sched.push_back((int16_t)((uint32_t)base >> 16));
            }
            // entries of the batch, structure-of-arrays: [e][slot]
            const int32_t cnt = bcount[j];
            const size_t s0 = sched.size(), v0 = vperm.size();
            sched.resize(s0 + (size_t)cnt * MD, (int16_t)zslot);  // padding: zero cell, zero factor
            vperm.resize(v0 + (size_t)cnt * MD, -1);              // (acc - 0 * 0 == acc exactly)
            for (int32_t u = 0; u < cnt; ++u) {
                const int32_t i = LS.h_rowof[bslot[j] + u];
                if (i < 0) continue;
                int32_t e = 0;
                auto push = [&](int32_t p) {
                    const int32_t jj = col[p];
                    const bool prev = line[jj] == line[i] && jj == i + (upper ? 1 : -1);
                    const int32_t pj = upper ? (starts[line[jj] + 1] - 1 - jj) : pos[jj];
#ifdef NPCG_LINE_AOS
                    const size_t at = (size_t)u * MD + e;
#else
                    const size_t at = (size_t)e * cnt + u;
#endif
                    sched[s0 + at] = (int16_t)(prev ? -1 : (pj & (W - 1)) * T + line[jj]);
                    vperm[v0 + at] = p;
                    ++e;
                };
                // the reference's summation order (sparse.py:222-239)
                if (upper)
                    for (int32_t p = rp[i + 1] - 1; p > dp[i]; --p) push(p);
                else
                    for (int32_t p = rp[i]; p < dp[i]; ++p) push(p);
            }
        }
        D.T = T;
        D.nbatch = nb;
        D.window = W;
        D.md = MD;
        D.zslot = zslot;
        D.max_slots = maxs;
        D.sched_words = (int64_t)sched.size();
        D.fac_slots = (int64_t)vperm.size();
        D.line_row0 = upload(row0);
        D.line_len = upload(llen);
        D.line_start = upload(lst);
        D.bslot = upload(db);
        D.bcount = upload(dc);
        D.boff = upload(boff);
        D.sched = upload(sched);
        D.vperm = upload(vperm);
        return D.line_row0 && D.line_len && D.line_start && D.bslot && D.bcount && D.boff && D.sched && D.vperm;
    };
    if (!build_dir(false, LS.fwd) || !build_dir(true, LS.bwd)) return false;
    LS.rowof = upload(LS.h_rowof);
    LS.slot = upload(LS.h_slot);
    return LS.rowof && LS.slot;
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
