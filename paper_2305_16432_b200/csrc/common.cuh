// common.cuh -- device helpers shared by the npcg kernels (internal).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace npcg {

constexpr int kMaxThresholds = 16;
constexpr int kMaxGroup = 32;  // columns per triangular-solve unit

int num_sms();
void keep_pool_memory();  // keep cudaMallocAsync scratch pooled across calls
void note_launch();  // launch accounting (npcg_launch_count)
long long launch_count();

// ---- memory-model helpers (PTX, gpu scope) --------------------------------
__device__ __forceinline__ int ld_acquire(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int *p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// ---- per-system PCG state (pcg.py:75-176 locals, one slot per column) ------
enum Status : int { ST_ACTIVE = 0, ST_CONVERGED = 1, ST_MAXITER = 2, ST_BREAKDOWN = 3 };
// Phase of an ACTIVE column inside the fixed kernel sequence of one pass:
//  PH_INIT    : this pass computes z = P^-1 r, p = z, rz = r.z (pcg.py:128-130,
//               and the restart branch pcg.py:161-165); k does not advance.
//  PH_ITER    : a regular iteration k -> k+1 (pcg.py:133-171).
//  PH_DRIFT   : recurrence residual crossed t_min; the drift kernel recomputes
//               b - A x (pcg.py:147-165).
//  PH_RESTART : drift found; skip the rest of this pass, next pass is PH_INIT.
enum Phase : int { PH_INIT = 0, PH_ITER = 1, PH_DRIFT = 2, PH_RESTART = 3 };
// What pupd does for a column at the end of a pass. PF_X: apply the pending
// x += alpha p of this pass first (the update is deferred out of the
// triangular solve; the drift check reads x + alpha p on the fly).
enum PFlag : int { PF_NONE = 0, PF_UPDATE = 1, PF_COPY = 2, PF_X = 4 };

struct SolveState {
    // per column [B]
    int *status, *phase, *pflag;
    int *xpend;                // 1 while this pass's x += alpha p is pending
    // line path: the x update runs as its own launch on a side stream, concurrent with the
    // P^{-1} launch (it needs alpha and p_k only). xgo[b] == epoch marks the columns whose
    // alpha this pass's SpMV formed; null: the update stays in pupd.
    int *xgo;
    int epoch;
    long long *k;              // iterations
    long long *breakdown_at;
    double *scale, *rz, *alpha, *beta, *rel, *final_rel;
    long long *iter_to;        // [B][T]
    unsigned long long *t_to;  // [B][T] globaltimer at crossing
    double *history;           // [B][cap]
    long long history_cap;
    // scalars
    unsigned long long *t_start;
    int *active_count;
    // options
    int T;
    double thr[kMaxThresholds];
    long long max_iter;
    int absolute;
};

// Reduction scratch + counters used by the "last block reduces" epilogues.
struct Ctl {
    int next_unit;   // dynamic unit counter (SpTRSV)
    int done;        // finished blocks / units
    int exited;      // CTAs that found no unit left
    int pad[29];     // keep controls of different kernels on separate lines
};

__device__ __forceinline__ void record(const SolveState &st, int b, long long k, double v) {
    // pcg.py:116-120: every threshold not yet crossed with v <= t.
    for (int t = 0; t < st.T; ++t) {
        long long *slot = st.iter_to + (size_t)b * st.T + t;
        if (*slot < 0 && v <= st.thr[t]) {
            *slot = k;
            st.t_to[(size_t)b * st.T + t] = globaltimer();
        }
    }
}

__device__ __forceinline__ void push_history(const SolveState &st, int b, long long k, double v) {
    if (k < st.history_cap) st.history[(size_t)b * st.history_cap + k] = v;
}

// Forward-solve epilogue: residual norm of the updated r (pcg.py:143-150, 166).
__device__ inline void fwd_epilogue(const SolveState &st, int b, double total, int *drift_count) {
    if (st.status[b] != ST_ACTIVE || st.phase[b] != PH_ITER) return;
    const double rn = sqrt(total);
    const long long k = st.k[b];
    push_history(st, b, k, rn);
    const double rel = rn / st.scale[b];
    st.rel[b] = rel;
    if (rel <= st.thr[st.T - 1]) {
        st.phase[b] = PH_DRIFT;
        atomicAdd(drift_count, 1);
    } else {
        record(st, b, k, rel);
    }
}

// Backward-solve epilogue: r.z and what pupd does next (pcg.py:128-130, 167-171).
__device__ inline void bwd_epilogue(const SolveState &st, int b, double total) {
    int f = PF_NONE;
    if (st.status[b] == ST_ACTIVE) {
        const int ph = st.phase[b];
        if (ph == PH_ITER) {
            st.beta[b] = total / st.rz[b];
            st.rz[b] = total;
            f = PF_UPDATE;
        } else if (ph == PH_INIT) {
            st.rz[b] = total;
            f = PF_COPY;
            st.phase[b] = PH_ITER;
        } else if (ph == PH_RESTART) {
            st.phase[b] = PH_INIT;
        }
    }
    if (st.xpend[b]) {  // converged, restarted or iterating: x_{k+1} = x_k + alpha p_k
        f |= PF_X;
        st.xpend[b] = 0;
    }
    st.pflag[b] = f;
}

}  // namespace npcg
