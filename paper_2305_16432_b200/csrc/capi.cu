// capi.cu -- extern "C" entry points of libnpcg.so (include/npcg.h).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/npcg.h"
#include "fem.cuh"
#include "train.cuh"

#include <nvtx3/nvToolsExt.h>  // header-only: ranges show up under Nsight tools, no-ops otherwise
#include "gnn.cuh"
#include "kernels.cuh"
#include "pattern.h"

using namespace npcg;

namespace {
// NVTX range over an entry point (the reference has no tracing; SURVEY.md section 5 lists it)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

struct npcg_pattern : public npcg::Pattern {
    // npcg_ldlt_apply_inverse workspaces by batch width (schedule packing,
    // scratch vectors): built once, reused by every later call; the mutex
    // serialises calls that share one
    std::mutex apply_mu;
    std::map<int, std::shared_ptr<npcg_solver>> apply_cache;
};

namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

#define NPCG_CUDA(call)                                                                   \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return fail(NPCG_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

template <class T>
cudaError_t dalloc(T **p, size_t count) {
    return cudaMalloc((void **)p, std::max<size_t>(count, 1) * sizeof(T));
}

// Pick the batch group width G (columns per unit) and chunk size for a solve.
struct SolvePlan {
    int G = 1, groups = 1, R = 1;
    SchedSet *set = nullptr;
};

// Columns per unit (G) and rows per chunk (R). G = 1 keeps every level's
// items on distinct rows and gives B independent pipelines; the shared-
// memory ring (window x level width x G doubles) must fit, otherwise the
// chunks are made smaller (narrower levels).
int plan_solve(Pattern *F, int B, SolvePlan &plan, std::string &err) {
    int G = 1;
    if (const char *env = std::getenv("NPCG_GROUP")) {
        int v = std::atoi(env);
        if (v >= 1 && v <= kMaxGroup && (v & (v - 1)) == 0) G = std::min(v, std::max(1, B));
    }
    if (B % 2) G = 1;  // 16-byte vector staging needs an even column stride
    int R = choose_chunk_rows(F->n, B, G);
    size_t cap = 200 * 1024;  // deep (3-D) level sets: longer chunks, fewer cross-chunk hand-offs (measured)
    if (const char *env = std::getenv("NPCG_SMEM_KB")) cap = (size_t)std::max(16, std::atoi(env)) * 1024;
    for (;;) {
        SchedSet *set = F->schedule(R, err);
        if (!set) return NPCG_ERR_CUDA;
        // worst case: batched factor values staged per column
        const size_t smem = std::max(trsv_smem_plan(set->fwd, G, 1).total, trsv_smem_plan(set->bwd, G, 1).total);
        if (smem <= cap || R <= 64) {
            if (smem > 220 * 1024) {
                err = "triangular-solve ring does not fit in shared memory";
                return NPCG_ERR_ARGUMENT;
            }
            plan.G = G;
            plan.groups = (B + G - 1) / G;
            plan.R = R;
            plan.set = set;
            if (std::getenv("NPCG_VERBOSE"))
                fprintf(stderr,
                        "[npcg] plan n=%lld B=%d G=%d R=%d chunks=%d units=%d | fwd maxw=%d words=%d se=%d x=%d "
                        "W=%d levels=%d | bwd maxw=%d W=%d | smem=%zu\n",
                        (long long)F->n, B, G, R, set->fwd.chunks, set->fwd.chunks * plan.groups, set->fwd.maxw,
                        set->fwd.max_words, set->fwd.max_se, set->fwd.maxx, set->fwd.window,
                        set->fwd.max_chunk_levels, set->bwd.maxw, set->bwd.window, smem);
            return NPCG_OK;
        }
        if (G > 1) G /= 2;
        else R = (R + 1) / 2;
    }
}

int check_stream_device() {
    int dev = 0, major = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return fail(NPCG_ERR_CUDA, "no CUDA device");
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    if (major != 10) return fail(NPCG_ERR_CUDA, "libnpcg is built for sm_100a (B200) only");
    return NPCG_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// solver workspace
// ---------------------------------------------------------------------------
struct npcg_solver {
    const Pattern *A = nullptr;
    Pattern *F = nullptr;
    std::unique_ptr<npcg_pattern> identity;  // when F == NULL
    int B = 1;
    SolvePlan plan;
    double *R = nullptr, *P = nullptr, *Z = nullptr, *AP = nullptr, *Y = nullptr;
    // state
    int *status = nullptr, *phase = nullptr, *pflag = nullptr;
    long long *k = nullptr, *bd = nullptr, *iter_to = nullptr;
    unsigned long long *t_to = nullptr, *t_start = nullptr;
    double *scale = nullptr, *rz = nullptr, *alpha = nullptr, *beta = nullptr, *rel = nullptr,
           *final_rel = nullptr;
    double *history = nullptr;
    long long history_cap = 0;
    int *active_count = nullptr, *drift_count = nullptr;
    Ctl *ctl = nullptr;
    double *partial = nullptr;
    double *S_fwd = nullptr, *S_bwd = nullptr;  // factor entries in schedule order
    size_t S_cap = 0;
    LineSched *ls = nullptr;  // line-wavefront schedule (owned by the pattern) or null
    LevelSched *lv = nullptr;  // global level sets for the level-synchronous kernel, or null
    unsigned *gbar = nullptr;  // its grid barrier words
    double *lpartial = nullptr;  // its per-block partial sums [grid][B]
    unsigned *lflags = nullptr;  // dependency-flag mode: [n][level_flag_groups(B)], or null (barrier per level)
    unsigned lepoch = 0;         // epoch of the last level launch
    int line_K = 0;  // launch shape (line_config_for) of the line P^{-1} kernel
    int line_KS = 0; // the same with several systems per cluster (shared factor only; 0: none)
    // line mode: every loop vector is in line order ([b][nslot]): P, XL (x), BL (b)
    // too; A as ELL by slot
    double *XL = nullptr, *BL = nullptr;
    int ell_width = 0;
    int *ecol = nullptr, *eperm = nullptr;  // [ell_width][nslot]: column slot / natural CSR position (-1: none)
    double *evals = nullptr;                // packed A values ([b][ell_width][nslot] or [ell_width][nslot])
    size_t evals_cap = 0, partial_cap = 0;
    double *Dl = nullptr, *rDl = nullptr;  // diag in line order ([b][nslot] or [nslot]) and 1 / diag
    size_t Dl_cap = 0;
    int *xpend = nullptr;
    int *xgo = nullptr;                    // line path: epoch of the pass whose x update is due (common.cuh)
    cudaStream_t side = nullptr;           // the x updates run here, beside the P^{-1} launch
    cudaEvent_t ev_spmv = nullptr, ev_x = nullptr;
    double *ones = nullptr;   // identity preconditioner: D = 1 (per solver: no shared state between threads)
    long long *kmax = nullptr;  // largest k of the batch at the last poll
    struct Poll {
        int active;
        int pad;
        long long kmax;
    };
    Poll *h_poll = nullptr;  // pinned, two slots (polls alternate)
    cudaEvent_t poll_ev[2] = {nullptr, nullptr};
    long long history_len = 0;  // entries per system valid after the last solve
    ~npcg_solver() {
        void *ptrs[] = {R, P, Z, AP, Y, status, phase, pflag, k, bd, iter_to, t_to, t_start, scale, rz,
                        alpha, beta, rel, final_rel, history, active_count, drift_count, ctl, partial,
                        S_fwd, S_bwd, xpend, Dl, rDl, XL, BL, ecol, eperm, evals, ones, kmax, gbar, lpartial, lflags};
        for (void *p : ptrs)
            if (p) cudaFree(p);
        if (h_poll) cudaFreeHost(h_poll);
        if (xgo) cudaFree(xgo);
        if (side) cudaStreamDestroy(side);
        if (ev_spmv) cudaEventDestroy(ev_spmv);
        if (ev_x) cudaEventDestroy(ev_x);
        for (cudaEvent_t e : poll_ev)
            if (e) cudaEventDestroy(e);
    }
};

extern "C" {

const char *npcg_last_error(void) { return g_err.c_str(); }
int npcg_abi_version(void) { return NPCG_ABI_VERSION; }

int npcg_device_ok(void) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) return 0;
    int dev = 0, major = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    return major == 10 ? 1 : 0;
}

// ---------------------------------------------------------------------------
int npcg_pattern_create(int64_t n, const int64_t *rp, const int64_t *col, int flags, npcg_pattern **out) {
    if (!out) return fail(NPCG_ERR_ARGUMENT, "out is NULL");
    *out = nullptr;
    if (n < 0 || !rp || (n > 0 && !col && rp[n] > 0))
        return fail(NPCG_ERR_DIMENSION, "row_ptr must have length n+1");
    // sparse.py:44-65 invariants
    if (rp[0] != 0) return fail(NPCG_ERR_DIMENSION, "row_ptr endpoints disagree with nnz");
    const int64_t nnz = rp[n];
    if (nnz >= (1ll << 31) || n >= (1ll << 31)) return fail(NPCG_ERR_DIMENSION, "pattern exceeds int32 indexing");
    for (int64_t i = 0; i < n; ++i)
        if (rp[i + 1] < rp[i]) return fail(NPCG_ERR_DIMENSION, "row_ptr must be non-decreasing");
    for (int64_t i = 0; i < n; ++i)
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
            if (col[p] < 0 || col[p] >= n) return fail(NPCG_ERR_DIMENSION, "column index out of range");
            if (p > rp[i] && col[p] <= col[p - 1])
                return fail(NPCG_ERR_DIMENSION, "columns must strictly increase within rows");
        }
    if (int rc = check_stream_device()) return rc;
    auto P = std::make_unique<npcg_pattern>();
    P->n = n;
    P->nnz = nnz;
    P->h_rp.assign(rp, rp + n + 1);
    P->h_col.assign(col, col + nnz);
    P->h_dp.assign(n, -1);
    P->h_pair.assign(nnz, -1);
    int64_t ndiag = 0, npair = 0;
    std::vector<int32_t> lower;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
            const int64_t j = col[p];
            if (j == i) {
                P->h_dp[i] = (int32_t)p;
                ++ndiag;
            }
            if (j < i) lower.push_back((int32_t)p);
            // reverse edge (j, i): binary search in row j (gnn.py:86-88)
            const int64_t *b0 = col + rp[j], *b1 = col + rp[j + 1];
            const int64_t *f = std::lower_bound(b0, b1, i);
            if (f != b1 && *f == i) {
                P->h_pair[p] = (int32_t)(f - col);
                ++npair;
            }
        }
    P->full_diag = ndiag == n;
    P->symmetric = npair == nnz;
    P->nnz_lower = (int64_t)lower.size();
    P->factor_ok = P->full_diag && P->symmetric;
    if ((flags & NPCG_PATTERN_FACTOR) && !P->full_diag)
        return fail(NPCG_ERR_DATA_FORMAT, "matrix is missing explicit diagonal entries");
    if ((flags & NPCG_PATTERN_FACTOR) && !P->symmetric)
        return fail(NPCG_ERR_DATA_FORMAT, "matrix pattern is not symmetric");
    NPCG_CUDA(dalloc(&P->rp, n + 1));
    NPCG_CUDA(dalloc(&P->col, nnz));
    NPCG_CUDA(dalloc(&P->dp, n));
    NPCG_CUDA(dalloc(&P->pair, nnz));
    NPCG_CUDA(dalloc(&P->lower_slot, lower.size()));
    NPCG_CUDA(dalloc(&P->src, nnz));
    {
        std::vector<int32_t> src(nnz);
        for (int64_t i = 0; i < n; ++i)
            for (int64_t p = rp[i]; p < rp[i + 1]; ++p) src[p] = (int32_t)i;
        if (nnz) NPCG_CUDA(cudaMemcpy(P->src, src.data(), nnz * 4, cudaMemcpyHostToDevice));
    }
    NPCG_CUDA(cudaMemcpy(P->rp, P->h_rp.data(), (n + 1) * 4, cudaMemcpyHostToDevice));
    if (nnz) NPCG_CUDA(cudaMemcpy(P->col, P->h_col.data(), nnz * 4, cudaMemcpyHostToDevice));
    if (n) NPCG_CUDA(cudaMemcpy(P->dp, P->h_dp.data(), n * 4, cudaMemcpyHostToDevice));
    if (nnz) NPCG_CUDA(cudaMemcpy(P->pair, P->h_pair.data(), nnz * 4, cudaMemcpyHostToDevice));
    if (!lower.empty())
        NPCG_CUDA(cudaMemcpy(P->lower_slot, lower.data(), lower.size() * 4, cudaMemcpyHostToDevice));
    *out = P.release();
    return NPCG_OK;
}

int npcg_pattern_destroy(npcg_pattern *p) {
    delete p;
    return NPCG_OK;
}

int npcg_pattern_get_info(const npcg_pattern *pc, npcg_pattern_info *info) {
    if (!pc || !info) return fail(NPCG_ERR_ARGUMENT, "NULL argument");
    npcg_pattern *p = const_cast<npcg_pattern *>(pc);
    std::memset(info, 0, sizeof(*info));
    info->n = p->n;
    info->nnz = p->nnz;
    info->nnz_lower = p->nnz_lower;
    info->full_diagonal = p->full_diag;
    info->structurally_symmetric = p->symmetric;
    info->has_factor_schedule = p->factor_ok;
    if (p->factor_ok) {  // report the most recently built schedule, if any (never builds one)
        std::lock_guard<std::mutex> lock(p->mu);
        if (p->scheds.empty()) return NPCG_OK;
        SchedSet *s = p->scheds.rbegin()->second.get();
        info->levels_lower = s->fwd.levels_global;
        info->levels_upper = s->bwd.levels_global;
        info->chunks = s->fwd.chunks;
        info->chunk_rows = s->fwd.chunk_rows;
        info->window = std::max(s->fwd.window, s->bwd.window);
        info->max_level_width = std::max(s->fwd.maxw, s->bwd.maxw);
    }
    return NPCG_OK;
}

int npcg_pattern_line_info(const npcg_pattern *pc, int32_t *lines, int32_t *warps, int32_t *steps, int32_t *cluster,
                           int batch) {
    if (!pc) return fail(NPCG_ERR_ARGUMENT, "NULL pattern");
    npcg_pattern *p = const_cast<npcg_pattern *>(pc);
    LineSched *ls = p->line_schedule();
    if (lines) *lines = ls ? ls->lines : 0;
    if (warps) *warps = ls ? ls->fwd.warps : 0;
    if (steps) *steps = ls ? ls->steps : 0;
    if (cluster) *cluster = ls ? line_cfg_cluster(line_config_for(*ls, std::max(batch, 1))) : 0;
    return NPCG_OK;
}

int npcg_pattern_device_arrays(const npcg_pattern *p, const int32_t **row_ptr, const int32_t **col_idx,
                               const int32_t **diag_pos, const int32_t **pair, const int32_t **lower_slot) {
    if (!p) return fail(NPCG_ERR_ARGUMENT, "NULL pattern");
    if (row_ptr) *row_ptr = p->rp;
    if (col_idx) *col_idx = p->col;
    if (diag_pos) *diag_pos = p->dp;
    if (pair) *pair = p->pair;
    if (lower_slot) *lower_slot = p->lower_slot;
    return NPCG_OK;
}

int npcg_check_symmetric_values(const npcg_pattern *p, int B, const double *vals, int vb, int32_t *ok_host,
                                void *stream) {
    if (!p || !ok_host || B < 1) return fail(NPCG_ERR_ARGUMENT, "bad argument");
    cudaStream_t s = (cudaStream_t)stream;
    for (int b = 0; b < B; ++b) ok_host[b] = p->symmetric ? 1 : 0;
    if (!p->symmetric || p->nnz == 0) return NPCG_OK;
    int *d_ok = nullptr;
    keep_pool_memory();
    NPCG_CUDA(cudaMallocAsync((void **)&d_ok, (size_t)B * 4, s));
    NPCG_CUDA(cudaMemcpyAsync(d_ok, ok_host, B * 4, cudaMemcpyHostToDevice, s));
    note_launch(); symmetric_check_kernel<<<std::min<long long>((p->nnz * B + 255) / 256, 4096), 256, 0, s>>>(p->nnz, B, vb,
                                                                                           p->pair, vals, d_ok);
    NPCG_CUDA(cudaGetLastError());
    NPCG_CUDA(cudaMemcpyAsync(ok_host, d_ok, B * 4, cudaMemcpyDeviceToHost, s));
    cudaFreeAsync(d_ok, s);
    NPCG_CUDA(cudaStreamSynchronize(s));
    return NPCG_OK;
}

// ---------------------------------------------------------------------------
int npcg_spmv(const npcg_pattern *A, int B, const double *vals, int vb, const double *x, double *y, void *stream) {
    NvtxRange nvtx_range("npcg_spmv");
    if (!A || B < 1 || B > kMaxBatch) return fail(NPCG_ERR_ARGUMENT, "bad pattern or batch");
    if (A->n == 0) return NPCG_OK;
    SpmvArgs a;
    a.n = (int)A->n;
    a.B = B;
    a.rp = A->rp;
    a.col = A->col;
    a.vals = vals;
    a.vb = vb;
    a.X = x;
    a.Y = y;
    a.op = SPMV_PLAIN;
    NPCG_CUDA(launch_spmv(a, (cudaStream_t)stream));
    return NPCG_OK;
}

int npcg_factor_from_lower(const npcg_pattern *F, int B, const double *lower, int lb, double *S, void *stream) {
    if (!F || B < 1) return fail(NPCG_ERR_ARGUMENT, "bad argument");
    if (!F->factor_ok) return fail(NPCG_ERR_DATA_FORMAT, "pattern cannot carry a factor");
    cudaStream_t s = (cudaStream_t)stream;
    if (F->nnz) NPCG_CUDA(cudaMemsetAsync(S, 0, (size_t)F->nnz * B * 8, s));
    if (F->nnz_lower) {
        const long long work = F->nnz_lower * (long long)B;
        note_launch(); factor_from_lower_kernel<<<(int)std::min<long long>((work + 255) / 256, 8192), 256, 0, s>>>(
            (int)F->nnz_lower, B, lb, F->lower_slot, F->pair, lower, S);
        NPCG_CUDA(cudaGetLastError());
    }
    return NPCG_OK;
}

int npcg_factor_to_lower(const npcg_pattern *F, int B, const double *S, double *lower, void *stream) {
    if (!F || B < 1) return fail(NPCG_ERR_ARGUMENT, "bad argument");
    if (F->nnz_lower) {
        const long long work = F->nnz_lower * (long long)B;
        note_launch(); factor_to_lower_kernel<<<(int)std::min<long long>((work + 255) / 256, 8192), 256, 0, (cudaStream_t)stream>>>(
            (int)F->nnz_lower, B, F->lower_slot, S, lower);
        NPCG_CUDA(cudaGetLastError());
    }
    return NPCG_OK;
}

static int make_identity_pattern(int64_t n, std::unique_ptr<npcg_pattern> &out) {
    std::vector<int64_t> rp(n + 1), col(n);
    for (int64_t i = 0; i <= n; ++i) rp[i] = i;
    for (int64_t i = 0; i < n; ++i) col[i] = i;
    npcg_pattern *p = nullptr;
    int rc = npcg_pattern_create(n, rp.data(), col.data(), NPCG_PATTERN_FACTOR, &p);
    out.reset(p);
    return rc;
}

// ---------------------------------------------------------------------------
int npcg_solver_create(const npcg_pattern *A, const npcg_pattern *F, int B, npcg_solver **out) {
    if (!A || !out || B < 1 || B > kMaxBatch) return fail(NPCG_ERR_ARGUMENT, "bad argument");
    if (F && F->n != A->n) return fail(NPCG_ERR_DIMENSION, "factor and matrix disagree on dimension");
    auto s = std::make_unique<npcg_solver>();
    s->A = A;
    s->B = B;
    if (F) {
        s->F = const_cast<npcg_pattern *>(F);
    } else {
        if (int rc = make_identity_pattern(A->n, s->identity)) return rc;
        s->F = s->identity.get();
    }
    std::string err;
    if (int rc = plan_solve(s->F, B, s->plan, err)) return fail(rc, err);
    if (LineSched *ls = s->F->line_schedule()) {
        const int k = line_config_for(*ls, B);
        if (k > 0) {
            s->ls = ls;
            s->line_K = k;
            // shared-factor batches may carry kr right-hand sides per cluster
            // (interleaved dependency chains, NPCG_LINE_KR = 2 / 4). Off by
            // default: at config 2 one right-hand side per 2-CTA cluster
            // already covers 128 SMs and the per-launch latency decides
            // (measured 123 us per 64 right-hand sides against 147 us with
            // kr = 2 on 4-CTA clusters); it pays when the batch exceeds the SMs.
            int kr = 1;
            if (const char *env = std::getenv("NPCG_LINE_KR")) kr = std::atoi(env);
            while (kr > 1 && !s->line_KS) {
                s->line_KS = line_config_for(*ls, B, kr);
                kr /= 2;
            }
        }
    }
    // without a line schedule: level-synchronous solves when the batch gives
    // every level enough rows x columns (NPCG_LEVELSYNC=0/1 forces)
    if (!s->ls) {
        bool use = (long long)A->n * B >= (1ll << 20);
        if (const char *env = std::getenv("NPCG_LEVELSYNC")) use = std::atoi(env) != 0;
        if (use) s->lv = s->F->level_schedule();
        if (s->lv) {
            NPCG_CUDA(dalloc(&s->gbar, 2));
            NPCG_CUDA(cudaMemset(s->gbar, 0, 8));
            NPCG_CUDA(dalloc(&s->lpartial, (size_t)std::max(1, level_sync_grid(B)) * B));
            // dependency flags instead of a grid barrier per level (NPCG_LEVELFLAGS=0: barriers)
            bool flags = true;
            if (const char *env = std::getenv("NPCG_LEVELFLAGS")) flags = std::atoi(env) != 0;
            if (flags) {
                const size_t words = (size_t)A->n * level_flag_groups(B);
                NPCG_CUDA(dalloc(&s->lflags, words));
                NPCG_CUDA(cudaMemset(s->lflags, 0, words * sizeof(unsigned)));
            }
        }
    }
    if (s->ls) {  // A as ELL by slot (the line-order loop); rows wider than 16 keep the level path
        const LineSched &ls = *s->ls;
        int width = 0;
        for (int64_t i = 0; i < A->n; ++i) width = std::max<int>(width, A->h_rp[i + 1] - A->h_rp[i]);
        s->ell_width = width <= 4 ? 4 : width <= 7 ? 7 : width <= 8 ? 8 : width <= 12 ? 12 : width <= 16 ? 16 : 0;
        if (!s->ell_width) s->ls = nullptr;
    }
    const size_t nB = (size_t)A->n * B;
    const size_t vB = s->ls ? (size_t)s->ls->nslot * B : nB;  // line-order vectors
    NPCG_CUDA(dalloc(&s->R, vB));
    NPCG_CUDA(dalloc(&s->P, vB));
    NPCG_CUDA(dalloc(&s->Z, vB));
    NPCG_CUDA(dalloc(&s->AP, vB));
    NPCG_CUDA(dalloc(&s->Y, vB));
    if (s->ls) {  // padding slots stay zero; A as ELL by slot for the SpMV
        NPCG_CUDA(dalloc(&s->XL, vB));
        NPCG_CUDA(dalloc(&s->BL, vB));
        for (double *v : {s->R, s->Z, s->AP, s->Y, s->P, s->XL, s->BL}) NPCG_CUDA(cudaMemset(v, 0, vB * 8));
        const LineSched &ls = *s->ls;
        const int E = s->ell_width;
        std::vector<int> ecol((size_t)E * ls.nslot, -1), eperm((size_t)E * ls.nslot, -1);
        for (int q = 0; q < ls.nslot; ++q) {
            const int i = ls.h_rowof[q];
            if (i < 0) continue;
            for (int p = A->h_rp[i], e = 0; p < A->h_rp[i + 1]; ++p, ++e) {  // the reference's row order
                ecol[(size_t)e * ls.nslot + q] = ls.h_slot[A->h_col[p]];
                eperm[(size_t)e * ls.nslot + q] = p;
            }
        }
        NPCG_CUDA(dalloc(&s->ecol, ecol.size()));
        NPCG_CUDA(dalloc(&s->eperm, eperm.size()));
        NPCG_CUDA(cudaMemcpy(s->ecol, ecol.data(), ecol.size() * 4, cudaMemcpyHostToDevice));
        NPCG_CUDA(cudaMemcpy(s->eperm, eperm.data(), eperm.size() * 4, cudaMemcpyHostToDevice));
    }
    NPCG_CUDA(dalloc(&s->status, B));
    NPCG_CUDA(dalloc(&s->xpend, B));
    if (s->ls) {  // x updates beside the P^{-1} launch (NPCG_XUPD_STREAM=0: inside pupd)
        bool on = true;
        if (const char *env = std::getenv("NPCG_XUPD_STREAM")) on = std::atoi(env) != 0;
        if (on) {
            NPCG_CUDA(dalloc(&s->xgo, B));
            NPCG_CUDA(cudaStreamCreateWithFlags(&s->side, cudaStreamNonBlocking));
            NPCG_CUDA(cudaEventCreateWithFlags(&s->ev_spmv, cudaEventDisableTiming));
            NPCG_CUDA(cudaEventCreateWithFlags(&s->ev_x, cudaEventDisableTiming));
        }
    }

    NPCG_CUDA(dalloc(&s->phase, B));
    NPCG_CUDA(dalloc(&s->pflag, B));
    NPCG_CUDA(dalloc(&s->k, B));
    NPCG_CUDA(dalloc(&s->bd, B));
    NPCG_CUDA(dalloc(&s->iter_to, (size_t)B * kMaxThresholds));
    NPCG_CUDA(dalloc(&s->t_to, (size_t)B * kMaxThresholds));
    NPCG_CUDA(dalloc(&s->t_start, 1));
    NPCG_CUDA(dalloc(&s->scale, B));
    NPCG_CUDA(dalloc(&s->rz, B));
    NPCG_CUDA(dalloc(&s->alpha, B));
    NPCG_CUDA(dalloc(&s->beta, B));
    NPCG_CUDA(dalloc(&s->rel, B));
    NPCG_CUDA(dalloc(&s->final_rel, B));
    NPCG_CUDA(dalloc(&s->active_count, 1));
    NPCG_CUDA(dalloc(&s->drift_count, 1));
    const int chunks = s->plan.set->fwd.chunks;
    const size_t units = (size_t)chunks * s->plan.groups;
    NPCG_CUDA(dalloc(&s->ctl, 1));
    NPCG_CUDA(cudaMemset(s->ctl, 0, sizeof(Ctl)));
    NPCG_CUDA(cudaMemset(s->drift_count, 0, 4));
    size_t part = std::max<size_t>((size_t)kReduceBlocksPerSm * num_sms() * B, units * s->plan.G);
    if (s->ls) part = std::max<size_t>(part, (size_t)((s->ls->nslot + kSpmvThreads - 1) / kSpmvThreads) * B);
    s->partial_cap = part;
    NPCG_CUDA(dalloc(&s->partial, part));
    NPCG_CUDA(dalloc(&s->kmax, 1));
    NPCG_CUDA(cudaMallocHost((void **)&s->h_poll, 2 * sizeof(npcg_solver::Poll)));
    for (cudaEvent_t &e : s->poll_ev) NPCG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    if (s->identity) {
        NPCG_CUDA(dalloc(&s->ones, A->n));
        std::vector<double> h(A->n, 1.0);
        if (A->n) NPCG_CUDA(cudaMemcpy(s->ones, h.data(), (size_t)A->n * 8, cudaMemcpyHostToDevice));
    }
    if (!s->ls) {  // level-kernel outputs start unsolved (sentinel), see trsv.cu
        launch_fill_sentinel((long long)nB, s->Y, 0);
        launch_fill_sentinel((long long)nB, s->Z, 0);
    }
    NPCG_CUDA(cudaDeviceSynchronize());
    *out = s.release();
    return NPCG_OK;
}

int npcg_solver_destroy(npcg_solver *s) {
    delete s;
    return NPCG_OK;
}

static SolveState make_state(npcg_solver *s, const npcg_solve_opts *o) {
    SolveState st{};
    st.status = s->status;
    st.xpend = s->xpend;
    st.xgo = s->xgo;
    st.epoch = 0;

    st.phase = s->phase;
    st.pflag = s->pflag;
    st.k = s->k;
    st.breakdown_at = s->bd;
    st.scale = s->scale;
    st.rz = s->rz;
    st.alpha = s->alpha;
    st.beta = s->beta;
    st.rel = s->rel;
    st.final_rel = s->final_rel;
    st.iter_to = s->iter_to;
    st.t_to = s->t_to;
    st.history = s->history;
    st.history_cap = s->history_cap;
    st.t_start = s->t_start;
    st.active_count = s->active_count;
    st.T = o->n_thresholds;
    for (int t = 0; t < o->n_thresholds; ++t) st.thr[t] = o->thresholds[t];
    st.max_iter = o->max_iter;
    st.absolute = o->absolute;
    return st;
}

// Gather the factor entries (CSR order, symmetric S) into each direction's
// schedule order; done once per solve call, not per iteration.
static int stage_factor(npcg_solver *s, const double *S, int sb, const double *D, int db, cudaStream_t st) {
    size_t need;
    if (s->ls) {
        need = (size_t)std::max(s->ls->fwd.fac_slots, s->ls->bwd.fac_slots) * (sb ? s->B : 1);
    } else if (s->lv) {
        need = (size_t)std::max<int64_t>(std::max(s->lv->fwd.entries, s->lv->bwd.entries), 1) * (sb ? s->B : 1);
    } else {
        const Schedule &f = s->plan.set->fwd, &b = s->plan.set->bwd;
        const size_t cols = sb ? (size_t)s->plan.groups * s->plan.G : 1;
        need = (size_t)std::max<int64_t>(std::max(f.padded_entries, b.padded_entries), 2) * cols;
    }
    if (need > s->S_cap) {
        if (s->S_fwd) cudaFree(s->S_fwd);
        if (s->S_bwd) cudaFree(s->S_bwd);
        s->S_fwd = s->S_bwd = nullptr;
        s->S_cap = 0;
        NPCG_CUDA(dalloc(&s->S_fwd, need));
        NPCG_CUDA(dalloc(&s->S_bwd, need));
        s->S_cap = need;
    }
    if (s->ls) {  // S batched is laid out S[p * B + b]
        launch_line_factor_pack(s->ls->fwd, s->B, sb, sb ? s->B : 1, 1, S, s->S_fwd, st);
        launch_line_factor_pack(s->ls->bwd, s->B, sb, sb ? s->B : 1, 1, S, s->S_bwd, st);
        // diag in line order; padding slots divide by one
        const size_t dneed = (size_t)s->ls->nslot * (db ? s->B : 1);
        if (dneed > s->Dl_cap) {
            if (s->Dl) cudaFree(s->Dl);
            if (s->rDl) cudaFree(s->rDl);
            s->Dl = s->rDl = nullptr;
            s->Dl_cap = 0;
            NPCG_CUDA(dalloc(&s->Dl, dneed));
            NPCG_CUDA(dalloc(&s->rDl, dneed));
            s->Dl_cap = dneed;
        }
        NPCG_CUDA(launch_to_line(s->ls->nslot, db ? s->B : 1, s->ls->rowof, D, db, 1.0, s->Dl, st));
        NPCG_CUDA(launch_reciprocal((long long)dneed, s->Dl, s->rDl, st));
    } else if (s->lv) {
        launch_level_factor_pack(s->lv->fwd.entries, s->B, sb, s->lv->fwd.sperm, S, s->S_fwd, st);
        launch_level_factor_pack(s->lv->bwd.entries, s->B, sb, s->lv->bwd.sperm, S, s->S_bwd, st);
    } else {
        launch_factor_pack(s->plan.set->fwd, s->B, s->plan.G, sb, S, s->S_fwd, st);
        launch_factor_pack(s->plan.set->bwd, s->B, s->plan.G, sb, S, s->S_bwd, st);
    }
    NPCG_CUDA(cudaGetLastError());
    return NPCG_OK;
}

// P^{-1} on the level path: one direction of the chunked level kernel.
// Vectors are RHS-minor (i*B + b).
static TrsvArgs level_args(npcg_solver *s, bool upper, int mode, int sb, const double *D, int db) {
    TrsvArgs v;
    const Pattern *F = s->F;
    v.n = (int)F->n;
    v.B = s->B;
    v.G = s->plan.G;
    v.groups = s->plan.groups;
    v.upper = upper;
    v.mode = mode;
    v.sched = upper ? s->plan.set->bwd : s->plan.set->fwd;
    v.units = v.sched.chunks * v.groups;
    v.S = upper ? s->S_bwd : s->S_fwd;
    v.s_batched = sb;
    v.D = D;
    v.d_batched = db;
    v.ctl = s->ctl;
    v.partial = s->partial;
    v.drift_count = s->drift_count;
    return v;
}

// one level launch; flag mode takes the next epoch (flags cleared before it wraps)
static cudaError_t level_launch(npcg_solver *s, LevelSyncArgs &a, cudaStream_t st) {
    if (a.flags) {
        if (s->lepoch == ~0u) {
            const cudaError_t e = cudaMemsetAsync(s->lflags, 0, (size_t)s->F->n * level_flag_groups(s->B) * sizeof(unsigned), st);
            if (e != cudaSuccess) return e;
            s->lepoch = 0;
        }
        a.epoch = ++s->lepoch;
    }
    return launch_level_sync(a, st);
}

static LevelSyncArgs level_sync_args(npcg_solver *s, bool upper, int mode, int sb, const double *D, int db) {
    LevelSyncArgs v;
    const LevelDir &L = upper ? s->lv->bwd : s->lv->fwd;
    v.B = s->B;
    v.upper = upper;
    v.mode = mode;
    v.nlev = L.nlev;
    v.lvl_ptr = L.lvl_ptr;
    v.rows = L.rows;
    v.eptr = L.eptr;
    v.ecol = L.ecol;
    v.S = upper ? s->S_bwd : s->S_fwd;
    v.s_batched = sb;
    v.D = D;
    v.d_batched = db;
    v.partial = s->lpartial;
    v.bar = s->gbar;
    v.flags = s->lflags;
    v.max_rows = L.max_rows;
    v.drift_count = s->drift_count;
    return v;
}

// P^{-1} on the line path: forward solve, y / D and backward solve in one
// launch (ldlt_line_kernel); every vector in line order ([b][nslot]).
static LineArgs line_args(npcg_solver *s, int mode, int sb, int db) {
    LineArgs l;
    const int cfg = (!sb && s->line_KS) ? s->line_KS : s->line_K;
    l.B = s->B;
    l.kr = std::max(1, cfg >> 16);
    l.cluster = line_cfg_cluster(cfg);
    l.group = cfg / 16 % 16;
    l.stages = cfg % 16;
    l.mode = mode;
    l.nslot = s->ls->nslot;
    l.warps = s->ls->fwd.warps;
    l.ring = std::max(s->ls->fwd.ring, s->ls->bwd.ring);
    l.meta_f = s->ls->fwd.meta;
    l.meta_b = s->ls->bwd.meta;
    l.fac_slots = s->ls->fwd.fac_slots;
    l.S_f = s->S_fwd;
    l.S_b = s->S_bwd;
    l.s_batched = sb;
    l.D = s->Dl;  // staged by stage_factor
    l.rD = s->rDl;
    l.d_batched = db;
    l.drift_count = s->drift_count;
    return l;
}

int npcg_ldlt_apply_inverse(const npcg_pattern *F, int B, const double *S, int sb, const double *D, int db,
                            const double *r, double *z, void *stream) {
    NvtxRange nvtx_range("npcg_ldlt_apply_inverse");
    if (!F || B < 1 || B > kMaxBatch) return fail(NPCG_ERR_ARGUMENT, "bad argument");
    if (!F->factor_ok) return fail(NPCG_ERR_DATA_FORMAT, "pattern cannot carry a factor");
    if (F->n == 0) return NPCG_OK;
    // a cached solver (per pattern and batch width) supplies the schedule,
    // scratch and counters
    npcg_pattern *Fm = const_cast<npcg_pattern *>(F);
    std::lock_guard<std::mutex> lock(Fm->apply_mu);
    std::shared_ptr<npcg_solver> &slot = Fm->apply_cache[B];
    if (!slot) {
        npcg_solver *made = nullptr;
        if (int rc = npcg_solver_create(F, F, B, &made)) {
            Fm->apply_cache.erase(B);
            return rc;
        }
        slot.reset(made, [](npcg_solver *p) { npcg_solver_destroy(p); });
    }
    npcg_solver *s = slot.get();
    cudaStream_t st = (cudaStream_t)stream;
    if (int rc = stage_factor(s, S, sb, D, db, st)) return rc;
    if (s->ls) {  // through line order: r -> R, (Y), Z -> z
        const LineSched &ls = *s->ls;
        NPCG_CUDA(launch_to_line(ls.nslot, B, ls.rowof, r, 1, 0.0, s->R, st));
        LineArgs l = line_args(s, TRSV_PLAIN, sb, db);
        l.in = s->R;
        l.Y = s->Y;
        l.out = s->Z;
        NPCG_CUDA(launch_ldlt_line(l, st));
        NPCG_CUDA(launch_from_line(ls.nslot, B, ls.rowof, s->Z, z, st));
    } else if (s->lv) {
        LevelSyncArgs f = level_sync_args(s, false, TRSV_PLAIN, sb, D, db);
        f.in = r;
        f.out = s->Y;
        NPCG_CUDA(level_launch(s, f, st));
        LevelSyncArgs b = level_sync_args(s, true, TRSV_PLAIN, sb, D, db);
        b.in = s->Y;
        b.out = z;
        NPCG_CUDA(level_launch(s, b, st));
    } else {
        launch_fill_sentinel((long long)F->n * B, z, st);  // level kernel polls z
        TrsvArgs f = level_args(s, false, TRSV_PLAIN, sb, D, db);
        f.in = const_cast<double *>(r);  // r is only read
        f.out = s->Y;
        NPCG_CUDA(launch_trsv(f, st));
        TrsvArgs b = level_args(s, true, TRSV_PLAIN, sb, D, db);
        b.in = s->Y;
        b.out = z;
        NPCG_CUDA(launch_trsv(b, st));
    }
    NPCG_CUDA(cudaStreamSynchronize(st));
    return NPCG_OK;
}

int npcg_pcg_solve(npcg_solver *s, const double *A_vals, int ab, const double *S, int sb, const double *D, int db,
                   const double *bvec, double *x, const double *x0, const npcg_solve_opts *o,
                   npcg_solve_report *rep, void *stream) {
    NvtxRange nvtx_range("npcg_pcg_solve");
    if (!s || !o || !rep || !bvec || !x) return fail(NPCG_ERR_ARGUMENT, "NULL argument");
    if (o->n_thresholds < 1 || o->n_thresholds > kMaxThresholds)
        return fail(NPCG_ERR_DIMENSION, "at least one threshold required");
    for (int t = 0; t < o->n_thresholds; ++t) {
        if (!(o->thresholds[t] > 0.0 && o->thresholds[t] < 1.0))
            return fail(NPCG_ERR_DIMENSION, "thresholds must lie in (0, 1)");
        if (t && !(o->thresholds[t] < o->thresholds[t - 1]))
            return fail(NPCG_ERR_DIMENSION, "thresholds must be strictly decreasing");
    }
    if (o->max_iter < 1) return fail(NPCG_ERR_DIMENSION, "max_iter must be at least 1");
    const int B = s->B, T = o->n_thresholds;
    const int n = (int)s->A->n;
    cudaStream_t st = (cudaStream_t)stream;
    const bool identity = s->identity != nullptr;
    // identity preconditioner: S unused, D = 1
    if (identity) {
        S = s->ones;  // never read: identity pattern has no off-diagonal entries
        sb = 0;
        D = s->ones;
        db = 0;
    }
    // history: [B][cap] on the device, grown on demand as iterations advance
    // (a history can reach max_iter + 1 entries, pcg.py:113,145, but rarely
    // does: it is not preallocated at that size)
    const bool want_hist = o->history != 0 || rep->history != nullptr;
    const long long hist_full = o->max_iter + 1;
    long long cap = want_hist ? std::min<long long>(hist_full, 1024) : 1;
    if (!s->history || s->history_cap < cap) {
        if (s->history) cudaFree(s->history);
        s->history = nullptr;
        s->history_cap = 0;
        NPCG_CUDA(dalloc(&s->history, (size_t)cap * B));
        s->history_cap = cap;
    } else {
        cap = want_hist ? std::min(hist_full, s->history_cap) : 1;
    }
    s->history_len = 0;
    SolveState sst = make_state(s, o);
    sst.history_cap = cap;
    if (n == 0) {
        for (int b = 0; b < B; ++b) {
            rep->status[b] = NPCG_STATUS_CONVERGED;
            rep->iterations[b] = 0;
        }
        return NPCG_OK;
    }
    const long long nB = (long long)n * B;
    const int ew_grid = (int)std::min<long long>((nB + 255) / 256, 4 * 1024);

    note_launch(); init_state_kernel<<<(B + 127) / 128, 128, 0, st>>>(sst, B, cap);
    NPCG_CUDA(cudaGetLastError());
    note_launch(); normb_kernel<<<std::min(kReduceBlocksPerSm * num_sms(), std::max(1, n / 64)), kSpmvThreads, 0, st>>>(
        n, B, bvec, sst, s->partial, s->ctl);
    NPCG_CUDA(cudaGetLastError());
    note_launch(); init_x_kernel<<<ew_grid, 256, 0, st>>>(nB, B, x0, x, sst);
    NPCG_CUDA(cudaGetLastError());

    SpmvArgs sp;
    sp.n = n;
    sp.B = B;
    sp.rp = s->A->rp;
    sp.col = s->A->col;
    sp.vals = A_vals;
    sp.vb = ab;
    sp.st = sst;
    sp.partial = s->partial;
    sp.ctl = s->ctl;
    sp.drift_count = s->drift_count;
    SpmvArgs spl = sp;  // PCG ops: every vector in line order
    double *xv = x;            // the iterate the loop updates
    const double *bv = bvec;
    if (s->ls) {
        const int ns = s->ls->nslot, E = s->ell_width;
        spl.n = ns;
        spl.nslot = ns;
        spl.ecol = s->ecol;
        spl.ell_width = E;
        spl.partial_cap = s->partial_cap;
        const size_t need = (size_t)E * ns * (ab ? B : 1);
        if (need > s->evals_cap) {
            if (s->evals) cudaFree(s->evals);
            s->evals = nullptr;
            s->evals_cap = 0;
            NPCG_CUDA(dalloc(&s->evals, need));
            s->evals_cap = need;
        }
        launch_gather_pack((long long)E * ns, B, ab, ab ? B : 1, 1, s->eperm, A_vals, s->evals, st);
        spl.evals = s->evals;
        NPCG_CUDA(launch_to_line(ns, B, s->ls->rowof, x, 1, 0.0, s->XL, st));
        NPCG_CUDA(launch_to_line(ns, B, s->ls->rowof, bvec, 1, 0.0, s->BL, st));
        xv = s->XL;
        bv = s->BL;
    }
    // r = b - A x0 (or b)
    SpmvArgs init = spl;
    init.op = SPMV_RESID_INIT;
    init.X = xv;
    init.Bv = bv;
    init.R = s->R;
    init.has_x = x0 != nullptr;
    NPCG_CUDA(launch_spmv(init, st));

    SpmvArgs apdot = spl;
    apdot.op = SPMV_APDOT;
    apdot.X = s->P;
    apdot.Y = s->AP;
    if (s->ls) {  // the drift check rides on the next APDOT launch (no separate drift SpMV)
        apdot.merge_drift = 1;
        apdot.X2 = xv;
        apdot.Bv = bv;
        apdot.R = s->R;
    }
    SpmvArgs drift = spl;
    drift.op = SPMV_RESID_DRIFT;
    drift.X = xv;
    drift.Bv = bv;
    drift.R = s->R;
    drift.P = s->P;
    // identity: S = ones is never referenced (no off-diagonal slots), packs to zeros
    if (int rc = stage_factor(s, S, sb, D, db, st)) return rc;
    if (!s->ls) {  // the level kernel's outputs start unsolved (re-armed every pass)
        launch_fill_sentinel(nB, s->Y, st);
        launch_fill_sentinel(nB, s->Z, st);
    }
    // P^{-1}: line path (one launch) or level path (forward, drift, backward)
    LineArgs ll{};
    TrsvArgs fw{}, bw{};
    LevelSyncArgs fwl{}, bwl{};
    if (s->lv) {
        fwl = level_sync_args(s, false, TRSV_PCG, sb, D, db);
        fwl.in = s->R;
        fwl.out = s->Y;
        fwl.R = s->R;
        fwl.AP = s->AP;
        fwl.st = sst;
        bwl = level_sync_args(s, true, TRSV_PCG, sb, D, db);
        bwl.in = s->Y;
        bwl.out = s->Z;
        bwl.R = s->R;
        bwl.st = sst;
    }
    if (s->ls) {
        ll = line_args(s, TRSV_PCG, sb, db);
        ll.in = s->R;
        ll.R = s->R;
        ll.AP = s->AP;
        ll.Y = s->Y;
        ll.out = s->Z;
        ll.st = sst;
    } else {
        fw = level_args(s, false, TRSV_PCG, sb, D, db);
        fw.in = s->R;
        fw.out = s->Y;
        fw.R = s->R;
        fw.AP = s->AP;
        fw.st = sst;
        bw = level_args(s, true, TRSV_PCG, sb, D, db);
        bw.in = s->Y;
        bw.out = s->Z;
        bw.R = s->R;
        bw.st = sst;
    }

    // Optional per-launch timing (npcg_solve_opts.profile): a start/stop
    // event pair around every launch of the loop, summed per kernel class.
    const bool prof = o->profile != 0;
    struct Ev {
        cudaEvent_t a, b;
        int slot;
    };
    std::vector<Ev> pool, used;
    double prof_ms[NPCG_PROF_SLOTS] = {0};
    long long prof_n[NPCG_PROF_SLOTS] = {0};
    auto timed = [&](int slot, auto &&launch) -> cudaError_t {
        if (!prof) return launch();
        Ev e;
        if (pool.empty()) {
            cudaEventCreate(&e.a);
            cudaEventCreate(&e.b);
        } else {
            e = pool.back();
            pool.pop_back();
        }
        e.slot = slot;
        cudaEventRecord(e.a, st);
        cudaError_t c = launch();
        cudaEventRecord(e.b, st);
        used.push_back(e);
        return c;
    };
    // NPCG_PROFILE_DUMP=<file>: also append every launch's (class, ms) (diagnostics)
    FILE *dump = nullptr;
    if (prof)
        if (const char *path = std::getenv("NPCG_PROFILE_DUMP")) dump = std::fopen(path, "a");
    auto harvest = [&]() {
        for (Ev &e : used) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e.a, e.b);
            prof_ms[e.slot] += ms;
            prof_n[e.slot] += 1;
            if (dump) std::fprintf(dump, "%d %.6f\n", e.slot, ms);
            pool.push_back(e);
        }
        used.clear();
    };
    auto pupd = [&]() {
        if (s->ls) return launch_pupd_ell(s->ls->nslot, B, s->Z, s->P, s->xgo ? nullptr : s->XL, sst, st);
        note_launch();
        pupd_kernel<<<ew_grid, 256, 0, st>>>(nB, B, s->Z, s->P, x, sst, 1);
        return cudaGetLastError();
    };

    // the kernels carry the state by value: refresh every copy after the
    // history buffer moved
    auto set_state = [&]() {
        apdot.st = drift.st = sst;
        fw.st = bw.st = ll.st = fwl.st = bwl.st = sst;
    };
    // Passes are enqueued in chunks of `check`; every chunk ends with a poll (active columns,
    // largest iteration count) copied to pinned memory and an event. The host waits for poll
    // k only after chunk k + 1 is enqueued, so the device never idles on the host; after the
    // last column converges at most one more chunk runs (every kernel takes its skip path).
    const int check = o->check_every > 0 ? o->check_every : 8;
    // a pass advances k by at most one; an iteration whose drift check
    // restarts takes three passes (iterate, restart, re-init)
    const long long max_passes = 3 * o->max_iter + 16;
    long long passes = 0;
    int epoch = 0;
    if (s->xgo) NPCG_CUDA(cudaMemsetAsync(s->xgo, 0, (size_t)B * sizeof(int), st));
    auto enqueue_chunk = [&]() -> int {
        for (int q = 0; q < check; ++q) {
            apdot.st.epoch = ++epoch;
            NPCG_CUDA(timed(NPCG_PROF_SPMV_APDOT, [&] { return launch_spmv(apdot, st); }));
            if (s->ls) {  // P^{-1} in one launch, then the p update; x += alpha p beside it
                if (s->xgo) {
                    NPCG_CUDA(cudaEventRecord(s->ev_spmv, st));
                    NPCG_CUDA(cudaStreamWaitEvent(s->side, s->ev_spmv, 0));
                    NPCG_CUDA(launch_xupd_ell(s->ls->nslot, B, s->P, s->XL, apdot.st, s->side));
                    NPCG_CUDA(cudaEventRecord(s->ev_x, s->side));
                }
                NPCG_CUDA(timed(NPCG_PROF_TRSV_FWD, [&] { return launch_ldlt_line(ll, st); }));
                if (s->xgo) NPCG_CUDA(cudaStreamWaitEvent(st, s->ev_x, 0));  // p_k is read until here
                NPCG_CUDA(timed(NPCG_PROF_PUPD, pupd));
                continue;
            }
            NPCG_CUDA(timed(NPCG_PROF_TRSV_FWD, [&] { return s->lv ? level_launch(s, fwl, st) : launch_trsv(fw, st); }));
            NPCG_CUDA(timed(NPCG_PROF_SPMV_DRIFT, [&] { return launch_spmv(drift, st); }));
            NPCG_CUDA(timed(NPCG_PROF_TRSV_BWD, [&] { return s->lv ? level_launch(s, bwl, st) : launch_trsv(bw, st); }));
            NPCG_CUDA(timed(NPCG_PROF_PUPD, pupd));
        }
        passes += check;
        return NPCG_OK;
    };
    auto enqueue_poll = [&](int slot, bool last) -> int {
        note_launch(); count_active_kernel<<<1, 256, 0, st>>>(sst, B, s->kmax, last ? 1 : 0);
        NPCG_CUDA(cudaMemcpyAsync(&s->h_poll[slot].active, s->active_count, 4, cudaMemcpyDeviceToHost, st));
        NPCG_CUDA(cudaMemcpyAsync(&s->h_poll[slot].kmax, s->kmax, 8, cudaMemcpyDeviceToHost, st));
        NPCG_CUDA(cudaEventRecord(s->poll_ev[slot], st));
        return NPCG_OK;
    };
    int polls = 0;          // polls enqueued
    bool last_sent = false;  // the poll that closes the pass budget is enqueued
    if (int rc = enqueue_chunk()) return rc;
    last_sent = passes >= max_passes;
    if (int rc = enqueue_poll(polls++ & 1, last_sent)) return rc;
    for (;;) {
        const bool more = !last_sent;
        if (more) {
            if (int rc = enqueue_chunk()) return rc;
            last_sent = passes >= max_passes;
            if (int rc = enqueue_poll(polls++ & 1, last_sent)) return rc;
        }
        const int wslot = (more ? polls - 2 : polls - 1) & 1;
        NPCG_CUDA(cudaEventSynchronize(s->poll_ev[wslot]));
        if (s->h_poll[wslot].active == 0 || !more) break;
        // the chunk in flight and the next one write history entries up to kmax + 2 check
        const long long need = std::min(hist_full, s->h_poll[wslot].kmax + 2 * (long long)check + 2);
        if (want_hist && need > cap) {
            NPCG_CUDA(cudaStreamSynchronize(st));  // the chunk in flight still writes the old buffer
            const long long ncap = std::min(hist_full, std::max(2 * cap, need));
            double *nh = nullptr;
            NPCG_CUDA(dalloc(&nh, (size_t)ncap * B));
            NPCG_CUDA(cudaMemcpy2DAsync(nh, (size_t)ncap * 8, s->history, (size_t)cap * 8, (size_t)cap * 8, B,
                                        cudaMemcpyDeviceToDevice, st));
            NPCG_CUDA(cudaStreamSynchronize(st));
            cudaFree(s->history);
            s->history = nh;
            s->history_cap = cap = ncap;
            sst.history = nh;
            sst.history_cap = ncap;
            set_state();
        }
    }
    NPCG_CUDA(cudaStreamSynchronize(st));
    harvest();
    for (Ev &e : pool) {
        cudaEventDestroy(e.a);
        cudaEventDestroy(e.b);
    }
    if (dump) std::fclose(dump);
    rep->passes = passes;
    if (rep->kernel_ms)
        for (int q = 0; q < NPCG_PROF_SLOTS; ++q) rep->kernel_ms[q] = prof_ms[q];
    if (rep->kernel_launches)
        for (int q = 0; q < NPCG_PROF_SLOTS; ++q) rep->kernel_launches[q] = prof_n[q];
    // report
    std::vector<int> status(B);
    NPCG_CUDA(cudaMemcpyAsync(status.data(), s->status, B * 4, cudaMemcpyDeviceToHost, st));
    NPCG_CUDA(cudaStreamSynchronize(st));
    bool any_max = false;
    for (int b = 0; b < B; ++b) any_max |= status[b] == ST_MAXITER || status[b] == ST_ACTIVE;
    if (any_max) {
        // columns still ACTIVE after the pass budget were turned into MAXITER
        SpmvArgs fin = spl;
        fin.op = SPMV_RESID_FINAL;
        fin.X = xv;
        fin.Bv = bv;
        NPCG_CUDA(launch_spmv(fin, st));
    }
    if (s->ls) NPCG_CUDA(launch_from_line(s->ls->nslot, B, s->ls->rowof, s->XL, x, st));
    std::vector<long long> kk(B), itto((size_t)B * T), bdv(B);
    std::vector<unsigned long long> tto((size_t)B * T);
    unsigned long long t0 = 0;
    NPCG_CUDA(cudaMemcpyAsync(kk.data(), s->k, B * 8, cudaMemcpyDeviceToHost, st));
    NPCG_CUDA(cudaMemcpyAsync(bdv.data(), s->bd, B * 8, cudaMemcpyDeviceToHost, st));
    NPCG_CUDA(cudaMemcpyAsync(itto.data(), s->iter_to, (size_t)B * T * 8, cudaMemcpyDeviceToHost, st));
    NPCG_CUDA(cudaMemcpyAsync(tto.data(), s->t_to, (size_t)B * T * 8, cudaMemcpyDeviceToHost, st));
    NPCG_CUDA(cudaMemcpyAsync(&t0, s->t_start, 8, cudaMemcpyDeviceToHost, st));
    NPCG_CUDA(cudaMemcpyAsync(rep->final_relative_residual, s->final_rel, B * 8, cudaMemcpyDeviceToHost, st));
    NPCG_CUDA(cudaStreamSynchronize(st));
    long long kmax = 0;
    for (int b = 0; b < B; ++b) {
        rep->status[b] = status[b] == ST_ACTIVE ? NPCG_STATUS_MAXITER : status[b];
        rep->iterations[b] = kk[b];
        if (rep->breakdown_iteration) rep->breakdown_iteration[b] = bdv[b];
        kmax = std::max(kmax, kk[b]);
        for (int t = 0; t < T; ++t) {
            rep->iterations_to[(size_t)b * T + t] = itto[(size_t)b * T + t];
            rep->seconds_to[(size_t)b * T + t] =
                itto[(size_t)b * T + t] >= 0 ? (double)(tto[(size_t)b * T + t] - t0) * 1e-9 : -1.0;
        }
    }
    s->history_len = want_hist ? std::min<long long>(kmax + 1, cap) : 0;
    if (rep->history) {
        const long long w = std::min<long long>(s->history_len, rep->history_cap);
        NPCG_CUDA(cudaMemcpy2DAsync(rep->history, (size_t)rep->history_cap * 8, s->history, (size_t)cap * 8,
                                    (size_t)w * 8, B, cudaMemcpyDeviceToHost, st));
        NPCG_CUDA(cudaStreamSynchronize(st));
    }
    return NPCG_OK;
}

int npcg_solver_history(const npcg_solver *s, double *out, int64_t ld, int64_t cols, void *stream) {
    if (!s || !out || ld < cols || cols < 0) return fail(NPCG_ERR_ARGUMENT, "bad argument");
    const long long w = std::min<long long>(cols, s->history_len);
    if (w <= 0) return NPCG_OK;
    cudaStream_t st = (cudaStream_t)stream;
    NPCG_CUDA(cudaMemcpy2DAsync(out, (size_t)ld * 8, s->history, (size_t)s->history_cap * 8, (size_t)w * 8, s->B,
                                cudaMemcpyDeviceToHost, st));
    NPCG_CUDA(cudaStreamSynchronize(st));
    return NPCG_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// GNN
// ---------------------------------------------------------------------------
struct npcg_gnn : public npcg::GnnDev {};

extern "C" {

int npcg_gnn_create(const npcg_gnn_desc *desc, const double *weights, int64_t n_weights, npcg_gnn **out) {
    if (!desc || !weights || !out) return fail(NPCG_ERR_ARGUMENT, "NULL argument");
    *out = nullptr;
    if (int rc = check_stream_device()) return rc;
    auto g = std::make_unique<npcg_gnn>();
    std::string err = gnn_init(*g, *desc, weights, n_weights);
    if (!err.empty()) return fail(NPCG_ERR_DIMENSION, err);
    *out = g.release();
    return NPCG_OK;
}

int npcg_gnn_destroy(npcg_gnn *g) {
    delete g;
    return NPCG_OK;
}

int npcg_gnn_build_factor(const npcg_gnn *g, const npcg_pattern *A, int B, const double *A_vals, int ab,
                          const double *rhs, double *S, double *D, double *edge_out, double *x0_out, int64_t *pivot,
                          void *stream) {
    NvtxRange nvtx_range("npcg_gnn_build_factor");
    if (!g || !A || !A_vals || !rhs || !S || !D || B < 1 || B > kMaxBatch) return fail(NPCG_ERR_ARGUMENT, "bad argument");
    if (g->d.north_star) return fail(NPCG_ERR_ARGUMENT, "north_star weights: use npcg_gnn_build_factor_mesh");
    if (!A->full_diag) return fail(NPCG_ERR_DATA_FORMAT, "matrix is missing explicit diagonal entries");
    if (!A->symmetric) return fail(NPCG_ERR_DATA_FORMAT, "matrix values are not symmetric");
    int64_t piv = -1;
    std::string err;
    const int rc = gnn_build(*g, *A, B, A_vals, ab, rhs, S, D, edge_out, x0_out, &piv, (cudaStream_t)stream, err);
    if (pivot) *pivot = piv;
    if (rc) return fail(rc, err);
    return NPCG_OK;
}

int npcg_gnn_build_factor_mesh(const npcg_gnn *g, const npcg_pattern *A, int B, const double *A_vals, int ab,
                               const double *rhs, const double *pos, const double *boundary, double *S, double *D,
                               double *edge_out, int64_t *pivot, void *stream) {
    NvtxRange nvtx_range("npcg_gnn_build_factor_mesh");
    if (!g || !A || !A_vals || !rhs || !S || !D || !pos || !boundary || B < 1 || B > kMaxBatch)
        return fail(NPCG_ERR_ARGUMENT, "bad argument");
    if (!g->d.north_star) return fail(NPCG_ERR_ARGUMENT, "reference weights: use npcg_gnn_build_factor");
    if (!A->full_diag) return fail(NPCG_ERR_DATA_FORMAT, "matrix is missing explicit diagonal entries");
    if (!A->symmetric) return fail(NPCG_ERR_DATA_FORMAT, "matrix values are not symmetric");
    GnnMesh mesh;
    mesh.pos = pos;
    mesh.boundary = boundary;
    int64_t piv = -1;
    std::string err;
    const int rc = gnn_build(*g, *A, B, A_vals, ab, rhs, S, D, edge_out, nullptr, &piv, (cudaStream_t)stream, err,
                             &mesh);
    if (pivot) *pivot = piv;
    if (rc) return fail(rc, err);
    return NPCG_OK;
}

}  // extern "C"

extern "C" int64_t npcg_launch_count(void) { return (int64_t)launch_count(); }

// ---------------------------------------------------------------------------
// Training step (train.cu): train.py:164-226 on the device
struct npcg_trainer {
    TrainNet net;
};

extern "C" int npcg_trainer_create(const npcg_gnn_desc *desc, const double *weights, int64_t n_weights,
                                   npcg_trainer **out) {
    if (!desc || !weights || !out) return fail(NPCG_ERR_ARGUMENT, "null argument");
    *out = nullptr;
    std::unique_ptr<npcg_trainer> t(new npcg_trainer);
    const std::string err = t->net.init(*desc, weights, n_weights);
    if (!err.empty()) return fail(NPCG_ERR_DIMENSION, err);
    *out = t.release();
    return NPCG_OK;
}

extern "C" int npcg_trainer_destroy(npcg_trainer *t) {
    delete t;
    return NPCG_OK;
}

extern "C" int npcg_trainer_get_weights(const npcg_trainer *t, double *weights_host) {
    if (!t || !weights_host) return fail(NPCG_ERR_ARGUMENT, "null argument");
    NPCG_CUDA(cudaMemcpy(weights_host, t->net.weights_dev(), (size_t)t->net.n_weights() * sizeof(double),
                         cudaMemcpyDeviceToHost));
    return NPCG_OK;
}

extern "C" int npcg_trainer_set_weights(npcg_trainer *t, const double *weights_host, int reset_moments) {
    if (!t || !weights_host) return fail(NPCG_ERR_ARGUMENT, "null argument");
    if (t->net.set_weights(weights_host, reset_moments)) return fail(NPCG_ERR_CUDA, "cudaMemcpy failed");
    return NPCG_OK;
}

extern "C" int npcg_trainer_tuple_grad(npcg_trainer *t, const npcg_pattern *A, const double *A_vals,
                                       const double *node_in, const double *edge_in, const double *b, const double *x,
                                       double x0_aux_weight, double *loss_host, double *grad_accum, void *stream) {
    NvtxRange nvtx_range("npcg_trainer_tuple_grad");
    if (!t || !A || !A_vals || !node_in || !edge_in || !b || !x || !loss_host || !grad_accum)
        return fail(NPCG_ERR_ARGUMENT, "null argument");
    std::string err;
    const int rc = t->net.tuple_grad(*A, A_vals, node_in, edge_in, b, x, x0_aux_weight, loss_host, grad_accum,
                                     (cudaStream_t)stream, err);
    return rc == NPCG_OK ? NPCG_OK : fail(rc, err);
}

extern "C" int npcg_trainer_adam_step(npcg_trainer *t, const double *grad, double grad_scale, int64_t step,
                                      double learning_rate, double beta1, double beta2, double eps, int32_t *nonfinite,
                                      void *stream) {
    if (!t || !grad || !nonfinite) return fail(NPCG_ERR_ARGUMENT, "null argument");
    if (step < 1) return fail(NPCG_ERR_DIMENSION, "Adam step index starts at 1");
    int nf = 0;
    const int rc = t->net.adam(grad, grad_scale, step, learning_rate, beta1, beta2, eps, &nf, (cudaStream_t)stream);
    *nonfinite = nf;
    return rc == NPCG_OK ? NPCG_OK : fail(rc, "CUDA failure in the Adam step");
}

// Restriction of assembled values to a sub-pattern (Dirichlet elimination,
// fem.py:209-215 / SparseMatrixCsr.submatrix): dst[q (* B + b)] = src[sel[q] (* B + b)].
extern "C" int npcg_gather_values(int64_t count, int B, int batched, const int32_t *sel, const double *src, double *dst,
                                  void *stream) {
    if (count < 0 || B < 1 || (count && (!sel || !src || !dst))) return fail(NPCG_ERR_ARGUMENT, "bad argument");
    if (count == 0) return NPCG_OK;
    // launch_gather_pack writes packed[b][e] = S[perm[e] * ps + b * bs]; with the
    // column index fastest on both sides one "system" of count * B entries does it
    cudaStream_t s = (cudaStream_t)stream;
    if (!batched || B == 1) {
        launch_gather_pack(count, 1, 0, 1, 0, sel, src, dst, s);
    } else {
        launch_gather_rows(count, B, sel, src, dst, s);
    }
    NPCG_CUDA(cudaGetLastError());
    return NPCG_OK;
}

// Diagnostics: the line-solve timeline of CTA 0 (clock64 per batch and event,
// [16][2048]); all zeros unless the library was built with -DNPCG_LINE_TRACE.
extern "C" int npcg_debug_line_trace(long long *out, int n) { return line_trace_copy(out, n); }

// ---- P1 FEM assembly (fem.cu) ---------------------------------------------
struct npcg_fem_plan {
    long long nv = 0, nt = 0, nnz = 0;
    int nper = 3;  // vertices per element
    std::vector<long long> row_ptr, col;
    int *d_starts = nullptr, *d_order = nullptr, *d_tri = nullptr;
    double *d_kq = nullptr, *d_ms = nullptr, *d_mq = nullptr;  // shared-mesh scratch (fem_prep_kernel)
};

extern "C" int npcg_fem_plan_create(int64_t nv, int64_t nt, const int64_t *tri, npcg_fem_plan **out) {
    return npcg_fem_plan_create_p1(nv, nt, 3, tri, out);
}

extern "C" int npcg_fem_plan_create_p1(int64_t nv, int64_t nt, int nper, const int64_t *tri, npcg_fem_plan **out) {
    if (!out || !tri) return fail(NPCG_ERR_ARGUMENT, "null argument");
    *out = nullptr;
    FemPlanHost h;
    const std::string err = fem_plan_build(nv, nt, nper, reinterpret_cast<const long long *>(tri), h);
    if (!err.empty()) return fail(NPCG_ERR_DATA_FORMAT, err);
    std::unique_ptr<npcg_fem_plan> p(new npcg_fem_plan);
    p->nv = nv;
    p->nt = nt;
    p->nper = nper;
    p->nnz = (long long)h.col.size();
    p->row_ptr = h.row_ptr;
    p->col.assign(h.col.begin(), h.col.end());
    std::vector<int> t32((size_t)nper * nt);
    for (long long q = 0; q < nper * nt; ++q) t32[q] = (int)tri[q];
    NPCG_CUDA(dalloc(&p->d_starts, h.starts.size()));
    NPCG_CUDA(dalloc(&p->d_order, h.order.size()));
    NPCG_CUDA(dalloc(&p->d_tri, t32.size()));
    NPCG_CUDA(dalloc(&p->d_kq, h.order.size()));
    NPCG_CUDA(dalloc(&p->d_ms, h.col.size()));
    NPCG_CUDA(dalloc(&p->d_mq, h.order.size()));
    NPCG_CUDA(cudaMemcpy(p->d_starts, h.starts.data(), h.starts.size() * 4, cudaMemcpyHostToDevice));
    NPCG_CUDA(cudaMemcpy(p->d_order, h.order.data(), h.order.size() * 4, cudaMemcpyHostToDevice));
    NPCG_CUDA(cudaMemcpy(p->d_tri, t32.data(), t32.size() * 4, cudaMemcpyHostToDevice));
    *out = p.release();
    return NPCG_OK;
}

extern "C" int npcg_fem_plan_destroy(npcg_fem_plan *p) {
    if (!p) return NPCG_OK;
    cudaFree(p->d_starts);
    cudaFree(p->d_order);
    cudaFree(p->d_tri);
    cudaFree(p->d_kq);
    cudaFree(p->d_ms);
    cudaFree(p->d_mq);
    delete p;
    return NPCG_OK;
}

extern "C" int npcg_fem_plan_pattern(const npcg_fem_plan *p, int64_t *nnz, int64_t *row_ptr, int64_t *col_idx) {
    if (!p || !nnz) return fail(NPCG_ERR_ARGUMENT, "null argument");
    *nnz = p->nnz;
    if (row_ptr) std::copy(p->row_ptr.begin(), p->row_ptr.end(), row_ptr);
    if (col_idx) std::copy(p->col.begin(), p->col.end(), col_idx);
    return NPCG_OK;
}

extern "C" int npcg_fem_assemble(const npcg_fem_plan *p, int B, const double *vertices, int vb, const double *coef,
                                 int cb, int mode, double scale, double *values, int *bad, void *stream) {
    NvtxRange nvtx_range("npcg_fem_assemble");
    if (!p || B < 1 || !vertices || !values) return fail(NPCG_ERR_ARGUMENT, "bad argument");
    if (mode != NPCG_FEM_K && mode != NPCG_FEM_M && mode != NPCG_FEM_M_PLUS_SK) return fail(NPCG_ERR_ARGUMENT, "bad mode");
    cudaStream_t s = (cudaStream_t)stream;
    int *flag = bad;
    if (!flag) {  // a scratch flag the caller does not read
        static thread_local int *scratch = nullptr;
        if (!scratch) NPCG_CUDA(dalloc(&scratch, 1));
        flag = scratch;
    }
    FemArgs a;
    a.nnz = (int)p->nnz;
    a.B = B;
    a.starts = p->d_starts;
    a.order = p->d_order;
    a.tri = p->d_tri;
    a.V = vertices;
    a.vb = vb ? B : 1;
    a.coef = coef;
    a.cb = cb ? B : 1;
    a.mode = mode;
    a.scale = scale;
    a.out = values;
    a.kq = p->d_kq;
    a.ms = p->d_ms;
    a.mq = p->d_mq;
    a.nt = (int)p->nt;
    a.nper2 = p->nper * p->nper;
    NPCG_CUDA(launch_fem_assemble(a, flag, s));
    return NPCG_OK;
}
