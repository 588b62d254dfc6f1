// kernels.cu -- sm_100a kernels of the PCG path: batched CSR SpMV with fused
// reductions, the chunked sync-free triangular solves, and the on-device PCG
// control logic (pcg.py:75-176) that runs inside "last block" epilogues so the
// host never synchronises per iteration.
//
// Arithmetic contract: every per-row sum uses the reference's summation
// order with explicitly unfused fp64 multiply / add (__dmul_rn, __dadd_rn),
// so spmv and ldlt_apply_inverse are bitwise identical to
// sparse.py:213-239; only dot products / norms (reductions) differ in
// order from numpy's BLAS ddot. Reductions are fixed-order (no float
// atomics), so the path is run-to-run deterministic.
#include <atomic>

#include "kernels.cuh"

namespace npcg {

// ===========================================================================
// SpMV family: Y = A X over a batch (vectors n x B, RHS-minor).
// A team of TL lanes owns one row; lane l handles columns l, l+TL, ...
// ===========================================================================

__device__ __forceinline__ bool spmv_col_active(const SpmvArgs &a, int b) {
    switch (a.op) {
        case SPMV_PLAIN: return true;
        case SPMV_APDOT:
            return a.st.status[b] == ST_ACTIVE && a.st.phase[b] == PH_ITER && a.st.k[b] < a.st.max_iter;
        case SPMV_RESID_INIT: return a.st.status[b] == ST_ACTIVE;
        case SPMV_RESID_DRIFT: return a.st.status[b] == ST_ACTIVE && a.st.phase[b] == PH_DRIFT;
        case SPMV_RESID_FINAL: return a.st.status[b] == ST_MAXITER;
    }
    return false;
}

// Per-column control logic after the batch reduction (one thread per column).
__device__ void spmv_epilogue(const SpmvArgs &a, int b, double total) {
    const SolveState &st = a.st;
    switch (a.op) {
        case SPMV_APDOT: {  // pcg.py:134-141
            if (st.status[b] != ST_ACTIVE || st.phase[b] != PH_ITER) return;
            if (st.k[b] >= st.max_iter) {  // while k < max_iter fell through
                st.status[b] = ST_MAXITER;
                return;
            }
            st.k[b] += 1;
            const double pAp = total;
            if (pAp <= 0.0) {  // BreakdownError; NaN passes like in numpy
                st.status[b] = ST_BREAKDOWN;
                st.breakdown_at[b] = st.k[b];
                return;
            }
            st.alpha[b] = st.rz[b] / pAp;
            st.xpend[b] = 1;  // x += alpha p happens in pupd (pcg.py:141)
            return;
        }
        case SPMV_RESID_INIT: {  // pcg.py:111-126
            if (st.status[b] != ST_ACTIVE) return;
            const double rn = sqrt(total);
            push_history(st, b, 0, rn);
            const double rel = rn / st.scale[b];
            st.rel[b] = rel;
            record(st, b, 0, rel);
            if (rel <= st.thr[st.T - 1]) {
                st.status[b] = ST_CONVERGED;
                st.final_rel[b] = rel;
            } else {
                st.phase[b] = PH_INIT;
            }
            return;
        }
        case SPMV_RESID_DRIFT: {  // pcg.py:147-165
            if (st.status[b] != ST_ACTIVE || st.phase[b] != PH_DRIFT) return;
            const double tn = sqrt(total);
            const double rel_t = tn / st.scale[b];
            const double rel = st.rel[b];
            const long long k = st.k[b];
            if (rel_t <= st.thr[st.T - 1]) {
                record(st, b, k, rel >= rel_t ? rel : rel_t);  // max(rel, rel_true)
                st.final_rel[b] = rel_t;
                st.status[b] = ST_CONVERGED;
            } else {
                record(st, b, k, rel_t);
                push_history(st, b, k, tn);  // history[-1] = ||r_true||
                st.rel[b] = rel_t;
                st.phase[b] = PH_RESTART;
            }
            return;
        }
        case SPMV_RESID_FINAL:  // pcg.py:171-172
            if (st.status[b] == ST_MAXITER) st.final_rel[b] = sqrt(total) / st.scale[b];
            return;
        default: return;
    }
}

template <int TL>
__global__ void __launch_bounds__(kSpmvThreads) spmv_kernel(SpmvArgs a) {
    constexpr int TEAMS = kSpmvThreads / TL;
    extern __shared__ double red[];  // TEAMS * B (reducing ops)
    __shared__ unsigned char s_act[kMaxBatch];
    __shared__ int s_last;
    const int team = threadIdx.x / TL, lane = threadIdx.x % TL;
    const int B = a.B;
    if (a.op == SPMV_RESID_DRIFT && *a.drift_count == 0) return;  // nothing drifted
    for (int b = threadIdx.x; b < B; b += blockDim.x) s_act[b] = spmv_col_active(a, b) ? 1 : 0;
    __syncthreads();
    const int cpl = (B + TL - 1) / TL;
    double part[kMaxCpl];
#pragma unroll
    for (int k = 0; k < kMaxCpl; ++k) part[k] = 0.0;

    for (int row = blockIdx.x * TEAMS + team; row < a.n; row += gridDim.x * TEAMS) {
        const int p0 = a.rp[row], p1 = a.rp[row + 1];
        double acc[kMaxCpl];
#pragma unroll
        for (int k = 0; k < kMaxCpl; ++k) acc[k] = 0.0;
        const bool use_x = a.op != SPMV_RESID_INIT || a.has_x;
        if (use_x) {
            for (int p = p0; p < p1; ++p) {
                const size_t j = (size_t)a.col[p] * B;
                const double vs = a.vb ? 0.0 : a.vals[p];
#pragma unroll
                for (int k = 0; k < kMaxCpl; ++k) {
                    const int b = lane + k * TL;
                    if (k < cpl && b < B) {
                        const double v = a.vb ? a.vals[(size_t)p * B + b] : vs;
                        double xv = a.X[j + b];
                        if (a.op == SPMV_RESID_DRIFT && a.st.xpend[b])  // x_{k+1} not yet stored
                            xv = __dadd_rn(xv, __dmul_rn(a.st.alpha[b], a.P[j + b]));
                        acc[k] = __dadd_rn(acc[k], __dmul_rn(v, xv));
                    }
                }
            }
        }
        const size_t ri = (size_t)row * B;
#pragma unroll
        for (int k = 0; k < kMaxCpl; ++k) {
            const int b = lane + k * TL;
            if (k >= cpl || b >= B || !s_act[b]) continue;
            switch (a.op) {
                case SPMV_PLAIN: a.Y[ri + b] = acc[k]; break;
                case SPMV_APDOT: {
                    a.Y[ri + b] = acc[k];
                    part[k] = __dadd_rn(part[k], __dmul_rn(a.X[ri + b], acc[k]));
                    break;
                }
                default: {  // residual r = b - A x
                    const double rt = __dsub_rn(a.Bv[ri + b], acc[k]);
                    if (a.op != SPMV_RESID_FINAL) a.R[ri + b] = rt;
                    part[k] = __dadd_rn(part[k], __dmul_rn(rt, rt));
                }
            }
        }
    }
    if (a.op == SPMV_PLAIN) return;

    // block reduction per column, fixed order over teams
#pragma unroll
    for (int k = 0; k < kMaxCpl; ++k) {
        const int b = lane + k * TL;
        if (k < cpl && b < B) red[team * B + b] = part[k];
    }
    __syncthreads();
    for (int b = threadIdx.x; b < B; b += blockDim.x) {
        double s = 0.0;
        for (int t = 0; t < TEAMS; ++t) s = __dadd_rn(s, red[t * B + b]);
        a.partial[(size_t)blockIdx.x * B + b] = s;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(&a.ctl->done, 1) == (int)gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // last block: grid reduction (fixed block order) + control epilogue
    const int G = gridDim.x;
    const int per = kSpmvThreads / (B < kSpmvThreads ? B : kSpmvThreads);  // threads per column
    double *scratch = red;  // reuse
    for (int b0 = 0; b0 < B; b0 += kSpmvThreads / per) {
        const int b = b0 + threadIdx.x / per, sub = threadIdx.x % per;
        double s = 0.0;
        if (b < B) {
            const int lo = (int)((long long)G * sub / per), hi = (int)((long long)G * (sub + 1) / per);
            for (int blk = lo; blk < hi; ++blk) s = __dadd_rn(s, __ldcg(&a.partial[(size_t)blk * B + b]));
        }
        scratch[threadIdx.x] = s;
        __syncthreads();
        if (sub == 0 && b < B) {
            double t = 0.0;
            for (int q = 0; q < per; ++q) t = __dadd_rn(t, scratch[threadIdx.x + q]);
            spmv_epilogue(a, b, t);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        a.ctl->done = 0;
        if (a.op == SPMV_RESID_DRIFT) *a.drift_count = 0;
    }
}

// ===========================================================================
// Elementwise / setup kernels
// ===========================================================================

__global__ void init_state_kernel(SolveState st, int B, long long hist_cap_init) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b == 0) *st.t_start = globaltimer();
    if (b >= B) return;
    st.status[b] = ST_ACTIVE;
    st.phase[b] = PH_INIT;
    st.pflag[b] = PF_NONE;
    st.xpend[b] = 0;
    st.k[b] = 0;
    st.breakdown_at[b] = 0;
    st.rz[b] = st.alpha[b] = st.beta[b] = st.rel[b] = st.final_rel[b] = 0.0;
    for (int t = 0; t < st.T; ++t) {
        st.iter_to[(size_t)b * st.T + t] = -1;
        st.t_to[(size_t)b * st.T + t] = 0;
    }
    (void)hist_cap_init;
}

// Column sums of squares of v (n x B) -> norm epilogue for ||b|| (pcg.py:93-102).
__global__ void __launch_bounds__(kSpmvThreads) normb_kernel(int n, int B, const double *v,
                                                              SolveState st, double *partial, Ctl *ctl) {
    __shared__ double red[kSpmvThreads];
    __shared__ int s_last;
    // thread -> (column b = tid % B', row offset) with B' = min(B, 256)
    const int cols = B < kSpmvThreads ? B : kSpmvThreads;
    const int rows_per = kSpmvThreads / cols;
    for (int b0 = 0; b0 < B; b0 += cols) {
        const int b = b0 + threadIdx.x % cols, r0 = threadIdx.x / cols;
        double s = 0.0;
        if (b < B && r0 < rows_per)
            for (long long i = (long long)blockIdx.x * rows_per + r0; i < n; i += (long long)gridDim.x * rows_per) {
                const double x = v[(size_t)i * B + b];
                s = __dadd_rn(s, __dmul_rn(x, x));
            }
        red[threadIdx.x] = s;
        __syncthreads();
        if (threadIdx.x < cols && b0 + threadIdx.x < B) {
            double t = 0.0;
            for (int q = 0; q < rows_per; ++q) t = __dadd_rn(t, red[q * cols + threadIdx.x]);
            partial[(size_t)blockIdx.x * B + b0 + threadIdx.x] = t;
        }
        __syncthreads();
    }
    __threadfence();
    if (threadIdx.x == 0) s_last = atomicAdd(&ctl->done, 1) == (int)gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (int b = threadIdx.x; b < B; b += blockDim.x) {
        double t = 0.0;
        for (int blk = 0; blk < (int)gridDim.x; ++blk) t = __dadd_rn(t, __ldcg(&partial[(size_t)blk * B + b]));
        const double nb = sqrt(t);
        if (nb == 0.0) {  // zero rhs: x = 0, 0 iterations, every threshold at 0
            st.status[b] = ST_CONVERGED;
            st.final_rel[b] = 0.0;
            push_history(st, b, 0, 0.0);
            const unsigned long long now = globaltimer();
            for (int q = 0; q < st.T; ++q) {
                st.iter_to[(size_t)b * st.T + q] = 0;
                st.t_to[(size_t)b * st.T + q] = now;
            }
        }
        st.scale[b] = st.absolute ? 1.0 : nb;
    }
    if (threadIdx.x == 0) ctl->done = 0;
}

// x = x0 (or 0); zero-rhs systems get x = 0 (pcg.py:95-101).
__global__ void init_x_kernel(long long nB, int B, const double *x0, double *x, SolveState st) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < nB; q += (long long)gridDim.x * blockDim.x) {
        const int b = (int)(q % B);
        x[q] = (x0 && st.status[b] == ST_ACTIVE) ? x0[q] : 0.0;
    }
}

// p = z + beta p  |  p = z   (pcg.py:129, 170)
__global__ void pupd_kernel(long long nB, int B, double *z, double *p, double *x, SolveState st, int rearm) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < nB; q += (long long)gridDim.x * blockDim.x) {
        const int b = (int)(q % B);
        const int f = st.pflag[b];
        if (f == PF_NONE) continue;
        const double pq = p[q];
        if (f & PF_X) x[q] = __dadd_rn(x[q], __dmul_rn(st.alpha[b], pq));  // pcg.py:141
        if (f & (PF_UPDATE | PF_COPY)) {
            const double zq = z[q];
            p[q] = (f & PF_UPDATE) ? __dadd_rn(zq, __dmul_rn(st.beta[b], pq)) : zq;  // pcg.py:129, 170
            if (rearm) reinterpret_cast<long long *>(z)[q] = (long long)kSentinel;  // for the next backward solve
        }
    }
}

__global__ void count_active_kernel(SolveState st, int B) {
    __shared__ int s;
    if (threadIdx.x == 0) s = 0;
    __syncthreads();
    for (int b = threadIdx.x; b < B; b += blockDim.x)
        if (st.status[b] == ST_ACTIVE) atomicAdd(&s, 1);
    __syncthreads();
    if (threadIdx.x == 0) *st.active_count = s;
}

// S[p] from strict-lower values in A.strict_lower() order (symmetric fill).
__global__ void factor_from_lower_kernel(int nnz_lower, int B, int lb, const int *lower_slot,
                                         const int *pair, const double *lower, double *S) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < (long long)nnz_lower * B;
         q += (long long)gridDim.x * blockDim.x) {
        const int s = (int)(q / B), b = (int)(q % B);
        const double v = lb ? lower[q] : lower[s];
        const int p = lower_slot[s];
        S[(size_t)p * B + b] = v;
        S[(size_t)pair[p] * B + b] = v;
    }
}

__global__ void factor_to_lower_kernel(int nnz_lower, int B, const int *lower_slot, const double *S,
                                       double *lower) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < (long long)nnz_lower * B;
         q += (long long)gridDim.x * blockDim.x) {
        const int s = (int)(q / B), b = (int)(q % B);
        lower[q] = S[(size_t)lower_slot[s] * B + b];
    }
}

// ok[b] &= vals[p] == vals[pair[p]] bitwise (sparse.py:137-147).
__global__ void symmetric_check_kernel(long long nnz, int B, int vb, const int *pair, const double *vals,
                                       int *ok) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < nnz * B;
         q += (long long)gridDim.x * blockDim.x) {
        const long long p = q / B;
        const int b = (int)(q % B);
        const int pp = pair[p];
        const double u = vb ? vals[q] : vals[p];
        const double v = vb ? vals[(size_t)pp * B + b] : vals[pp];
        if (__double_as_longlong(u) != __double_as_longlong(v)) ok[b] = 0;
    }
}

// ===========================================================================
// host launch helpers
// ===========================================================================

static std::atomic<long long> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
long long launch_count() { return g_launches.load(std::memory_order_relaxed); }

int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

static int team_lanes(int B) {
    int tl = 1;
    while (tl < B && tl < 32) tl <<= 1;
    return tl;
}

cudaError_t launch_spmv(const SpmvArgs &a, cudaStream_t s) {
    const int TL = team_lanes(a.B);
    const int teams = kSpmvThreads / TL;
    long long need = (a.n + teams - 1) / teams;
    int grid;
    if (a.op == SPMV_PLAIN) grid = (int)std::min<long long>(std::max<long long>(need, 1), 65535);
    else grid = (int)std::min<long long>(std::max<long long>(need, 1), (long long)kReduceBlocksPerSm * num_sms());
    size_t smem = a.op == SPMV_PLAIN ? 0 : (size_t)teams * a.B * sizeof(double);
    smem = std::max(smem, (size_t)kSpmvThreads * sizeof(double));
#define NPCG_SPMV_CASE(T)                                                                     \
    case T:                                                                                   \
        if (smem > 48 * 1024)                                                                 \
            cudaFuncSetAttribute(spmv_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                 (int)smem);                                                  \
        note_launch(); spmv_kernel<T><<<grid, kSpmvThreads, smem, s>>>(a);                                   \
        break;
    switch (TL) {
        NPCG_SPMV_CASE(1)
        NPCG_SPMV_CASE(2)
        NPCG_SPMV_CASE(4)
        NPCG_SPMV_CASE(8)
        NPCG_SPMV_CASE(16)
        NPCG_SPMV_CASE(32)
    }
#undef NPCG_SPMV_CASE
    return cudaGetLastError();
}

}  // namespace npcg
