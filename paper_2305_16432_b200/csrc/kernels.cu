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
#include <cstdlib>
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
            if (a.merge_drift && a.st.status[b] == ST_ACTIVE && a.st.phase[b] == PH_DRIFT) return true;
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
    const int op = (a.op == SPMV_APDOT && a.merge_drift && st.status[b] == ST_ACTIVE && st.phase[b] == PH_DRIFT)
                       ? SPMV_RESID_DRIFT
                       : a.op;
    switch (op) {
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
            if (st.xgo) st.xgo[b] = st.epoch;  // ... or in this pass's xupd launch
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

// X columns are read VW at a time (VW = 2: 16-byte loads when B is even).
// Row entries are consumed in groups of CH: all column indices of a group
// first, then all the X rows they name, so a team keeps CH independent
// loads in flight instead of a col -> x dependency per entry; products are
// still accumulated in entry order (bitwise the reference's row sum).
// Teams of >= 8 lanes own a contiguous block of rows: lane l holds entry
// p0 + l of the current row (one coalesced load, broadcast by shuffles) and
// the next row's entries are fetched while the current row's X loads fly.
template <int VW>
struct VecT;
template <>
struct VecT<1> {
    using type = double;
    static __device__ __forceinline__ void get(type v, double *o) { o[0] = v; }
};
template <>
struct VecT<2> {
    using type = double2;
    static __device__ __forceinline__ void get(type v, double *o) {
        o[0] = v.x;
        o[1] = v.y;
    }
};
template <>
struct VecT<4> {  // two 16-byte loads
    struct type {
        double2 lo, hi;
    };
    static __device__ __forceinline__ void get(const type &v, double *o) {
        o[0] = v.lo.x;
        o[1] = v.lo.y;
        o[2] = v.hi.x;
        o[3] = v.hi.y;
    }
};

// Row epilogue for one VW-column slot: store / fused dot / residual.
template <int VW>
__device__ __forceinline__ void spmv_row_pre(const SpmvArgs &a, size_t ri, int b, double *own) {
    // the row's own operand (p for p.Ap, b for r = b - Ax), loaded before the
    // row's sum so its latency overlaps the gathers
#pragma unroll
    for (int v = 0; v < VW; ++v)
        own[v] = a.op == SPMV_APDOT ? a.X[ri + b + v] : (a.op == SPMV_PLAIN ? 0.0 : a.Bv[ri + b + v]);
}

template <int VW>
__device__ __forceinline__ void spmv_row_out(const SpmvArgs &a, size_t ri, int b, const double *acc,
                                             const double *own, const unsigned char *s_act, double *pt) {
#pragma unroll
    for (int v = 0; v < VW; ++v) {
        const int bv = b + v;
        if (!s_act[bv]) continue;
        switch (a.op) {
            case SPMV_PLAIN: a.Y[ri + bv] = acc[v]; break;
            case SPMV_APDOT: {
                a.Y[ri + bv] = acc[v];
                pt[v] = __dadd_rn(pt[v], __dmul_rn(own[v], acc[v]));
                break;
            }
            default: {  // residual r = b - A x
                const double rt = __dsub_rn(own[v], acc[v]);
                if (a.op != SPMV_RESID_FINAL) a.R[ri + bv] = rt;
                pt[v] = __dadd_rn(pt[v], __dmul_rn(rt, rt));
            }
        }
    }
}

// acc += vals[e] * x[col[e]] over CH entries whose columns are in jj (-1 = none).
template <int CH, int VW, bool VB>
__device__ __forceinline__ void spmv_group(const SpmvArgs &a, const int *jj, const double *vs, int e0, int b,
                                           bool drift, const bool *xp, const double *al, double *acc) {
    using V = typename VecT<VW>::type;
    const int B = a.B;
    double vv[VB ? CH : 1][VW], xv[CH][VW];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        if (jj[c] < 0) continue;
        const size_t j = (size_t)jj[c] * B + b;
        if constexpr (VB) VecT<VW>::get(*reinterpret_cast<const V *>(a.vals + (size_t)(e0 + c) * B + b), vv[c]);
        VecT<VW>::get(*reinterpret_cast<const V *>(a.X + j), xv[c]);
        if (drift) {  // x_{k+1} = x + alpha p not yet stored (pcg.py:141)
            double pv[VW];
            VecT<VW>::get(*reinterpret_cast<const V *>(a.P + j), pv);
#pragma unroll
            for (int v = 0; v < VW; ++v)
                if (xp[v]) xv[c][v] = __dadd_rn(xv[c][v], __dmul_rn(al[v], pv[v]));
        }
    }
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        if (jj[c] < 0) continue;
#pragma unroll
        for (int v = 0; v < VW; ++v) acc[v] = __dadd_rn(acc[v], __dmul_rn(VB ? vv[VB ? c : 0][v] : vs[c], xv[c][v]));
    }
}

// Block reduction per column (fixed order over teams), then a grid reduction
// in fixed block order by the last block to finish, which runs the control
// epilogue. `red` holds [teams][ldr] partials of columns [b_lo, b_hi) (a
// 2-D grid splits the columns over blockIdx.y; rows of `partial` are
// blockIdx.x).
__device__ __forceinline__ void spmv_reduce_tail(const SpmvArgs &a, double *red, int teams, int b_lo = 0,
                                                 int b_hi = -1, int ldr = -1) {
    __shared__ int s_last;
    const int B = a.B;
    if (b_hi < 0) b_hi = B;
    if (ldr < 0) ldr = B;
    __syncthreads();
    for (int b = b_lo + threadIdx.x; b < b_hi; b += blockDim.x) {
        double s = 0.0;
        for (int t = 0; t < teams; ++t) s = __dadd_rn(s, red[t * ldr + b - b_lo]);
        a.partial[(size_t)blockIdx.x * B + b] = s;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(&a.ctl->done, 1) == (int)(gridDim.x * gridDim.y) - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const int G = gridDim.x;
    const int per = kSpmvThreads / (B < kSpmvThreads ? B : kSpmvThreads);  // threads per column
    double *scratch = red;  // reuse
    for (int b0 = 0; b0 < B; b0 += kSpmvThreads / per) {
        const int b = b0 + threadIdx.x / per, sub = threadIdx.x % per;
        double s = 0.0;
        if (b < B) {
            const int lo = (int)((long long)G * sub / per), hi = (int)((long long)G * (sub + 1) / per);
            int blk = lo;
            for (; blk + 8 <= hi; blk += 8) {  // 8 loads in flight, summed in block order
                double v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = __ldcg(&a.partial[(size_t)(blk + u) * B + b]);
#pragma unroll
                for (int u = 0; u < 8; ++u) s = __dadd_rn(s, v[u]);
            }
            for (; blk < hi; ++blk) s = __dadd_rn(s, __ldcg(&a.partial[(size_t)blk * B + b]));
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

template <int TL, int VW, bool VB>
__global__ void __launch_bounds__(kSpmvThreads, 2) spmv_kernel(SpmvArgs a) {
    constexpr int TEAMS = kSpmvThreads / TL, CH = 8;
    extern __shared__ double red[];  // TEAMS * B (reducing ops)
    __shared__ unsigned char s_act[kMaxBatch];
    const int team = threadIdx.x / TL, lane = threadIdx.x % TL;
    const int B = a.B;
    if (a.op == SPMV_RESID_DRIFT && *a.drift_count == 0) return;  // nothing drifted
    for (int b = threadIdx.x; b < B; b += blockDim.x) s_act[b] = spmv_col_active(a, b) ? 1 : 0;
    __syncthreads();
    const int cpl = (B + TL * VW - 1) / (TL * VW);  // VW-column slots per lane
    // per-(team, column) partial sums live in shared memory; each is owned by
    // one lane, so they accumulate in a fixed order without atomics
    double *part = red + team * B;
    if (a.op != SPMV_PLAIN)
        for (int b = lane; b < B; b += TL) part[b] = 0.0;
    const bool use_x = a.op != SPMV_RESID_INIT || a.has_x;
    const bool drift = a.op == SPMV_RESID_DRIFT;
    // per-slot drift state
    auto drift_state = [&](int b, bool *xp, double *al) {
#pragma unroll
        for (int v = 0; v < VW; ++v) {
            xp[v] = drift && a.st.xpend[b + v];
            al[v] = xp[v] ? a.st.alpha[b + v] : 0.0;
        }
    };

    if constexpr (TL >= CH) {
        // Entry stream: a team owns rows [r0, r1) and walks their entries
        // [rp[r0], rp[r1]) in windows of TL (lane l holds entry w + l, one
        // coalesced load), gathering CH X rows at a time regardless of where
        // rows end; a row's result is emitted when the stream crosses its end.
        const unsigned tmask = TL == 32 ? 0xffffffffu : (((1u << TL) - 1u) << ((threadIdx.x & 31) & ~(TL - 1)));
        const int nteams = gridDim.x * TEAMS, gteam = blockIdx.x * TEAMS + team;
        const int per = (a.n + nteams - 1) / nteams;
        const int r0 = min(a.n, gteam * per), r1 = min(a.n, r0 + per);
        if (r0 < r1) {
#pragma unroll 1
            for (int k = 0; k < cpl; ++k) {
                const int b = (lane + k * TL) * VW;
                const bool on = b < B;
                const int bb = on ? b : 0;
                bool xp[VW];
                double al[VW];
                drift_state(bb, xp, al);
                int row = r0, wb = r0 + 1;                   // rp window: rpl = rp[wb + lane]
                int rpl = a.rp[min(wb + lane, a.n)];
                int wi = 0;                                  // window index of row's end
                int rend = __shfl_sync(tmask, rpl, 0, TL);   // rp[row + 1]
                const int E0 = a.rp[r0];
                const int E1 = __shfl_sync(tmask, a.rp[r1], 0, TL);
                double acc[VW], own[VW];
#pragma unroll
                for (int v = 0; v < VW; ++v) acc[v] = 0.0;
                spmv_row_pre<VW>(a, (size_t)row * B, bb, own);
                // close row (store / dot) and open the next one
                auto next_row = [&]() {
                    if (on) spmv_row_out<VW>(a, (size_t)row * B, b, acc, own, s_act, part + b);
                    ++row;
#pragma unroll
                    for (int v = 0; v < VW; ++v) acc[v] = 0.0;
                    if (row < r1) {
                        spmv_row_pre<VW>(a, (size_t)row * B, bb, own);
                        if (++wi == TL) {
                            wb = row + 1;
                            rpl = a.rp[min(wb + lane, a.n)];
                            wi = 0;
                        }
                        rend = __shfl_sync(tmask, rpl, wi, TL);
                    }
                };
                if (use_x) {
                    for (int w = E0; w < E1; w += TL) {
                        const int cnt = min(TL, E1 - w);
                        const int cj = lane < cnt ? a.col[w + lane] : 0;
                        const double cv = (!VB && lane < cnt) ? a.vals[w + lane] : 0.0;
                        for (int g = 0; g < cnt; g += CH) {
                            using V = typename VecT<VW>::type;
                            double xv[CH][VW], vs[CH];
                            double vv[VB ? CH : 1][VW];
#pragma unroll
                            for (int c = 0; c < CH; ++c) {
                                const int j = __shfl_sync(tmask, cj, g + c, TL);
                                vs[c] = __shfl_sync(tmask, cv, g + c, TL);
                                if (g + c < cnt && on) {
                                    const size_t jo = (size_t)j * B + b;
                                    VecT<VW>::get(*reinterpret_cast<const V *>(a.X + jo), xv[c]);
                                    if constexpr (VB)
                                        VecT<VW>::get(*reinterpret_cast<const V *>(a.vals + (size_t)(w + g + c) * B + b), vv[c]);
                                    if (drift) {  // x_{k+1} = x + alpha p not yet stored (pcg.py:141)
                                        double pv[VW];
                                        VecT<VW>::get(*reinterpret_cast<const V *>(a.P + jo), pv);
#pragma unroll
                                        for (int v = 0; v < VW; ++v)
                                            if (xp[v]) xv[c][v] = __dadd_rn(xv[c][v], __dmul_rn(al[v], pv[v]));
                                    }
                                }
                            }
#pragma unroll
                            for (int c = 0; c < CH; ++c) {
                                const int ee = w + g + c;
                                if (ee >= E1) break;
                                while (ee == rend) next_row();  // rows ending before entry ee (incl. empty)
#pragma unroll
                                for (int v = 0; v < VW; ++v)
                                    acc[v] = __dadd_rn(acc[v], __dmul_rn(VB ? vv[VB ? c : 0][v] : vs[c], xv[c][v]));
                            }
                        }
                    }
                }
                while (row < r1) next_row();  // last row and trailing empty rows (or x = 0)
            }
        }
    } else {
        for (int row = blockIdx.x * TEAMS + team; row < a.n; row += gridDim.x * TEAMS) {
            const int p0 = a.rp[row], p1 = a.rp[row + 1];
            const size_t ri = (size_t)row * B;
#pragma unroll 1
            for (int k = 0; k < cpl; ++k) {
                const int b = (lane + k * TL) * VW;
                if (b >= B) continue;
                double acc[VW], own[VW];
#pragma unroll
                for (int v = 0; v < VW; ++v) acc[v] = 0.0;
                spmv_row_pre<VW>(a, ri, b, own);
                if (use_x) {
                    bool xp[VW];
                    double al[VW];
                    drift_state(b, xp, al);
                    for (int pb = p0; pb < p1; pb += CH) {
                        int jj[CH];
                        double vs[CH];
#pragma unroll
                        for (int c = 0; c < CH; ++c) {
                            jj[c] = pb + c < p1 ? a.col[pb + c] : -1;
                            vs[c] = (pb + c < p1 && !VB) ? a.vals[pb + c] : 0.0;
                        }
                        spmv_group<CH, VW, VB>(a, jj, vs, pb, b, drift, xp, al, acc);
                    }
                }
                spmv_row_out<VW>(a, ri, b, acc, own, s_act, part + b);
            }
        }
    }
    if (a.op == SPMV_PLAIN) return;

    spmv_reduce_tail(a, red, TEAMS);
}

// Warp-per-row SpMV for batches of >= 33 column groups (the common case,
// B >= 64 RHS): one warp owns a contiguous block of rows and handles one row
// per iteration with every lane covering VW adjacent columns, so a row's
// entries are one coalesced index load (lane l = entry l, broadcast by
// shuffles) and its gathers are CH unconditional 16-byte loads (padding
// slots re-read the row's own X row; their products are masked out of the
// sum). The op is a template parameter so the row loop has no switch, and
// the next row's indices are fetched while the current row's gathers fly.
template <int VW, bool VB, int OP>
__global__ void __launch_bounds__(kSpmvThreads, 2) spmv_warp_kernel(SpmvArgs a) {
    constexpr int TEAMS = kSpmvThreads / 32, CH = 8;
    using V = typename VecT<VW>::type;
    extern __shared__ double red[];  // TEAMS * B
    __shared__ unsigned char s_act[kMaxBatch];
    const int team = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int B = a.B;
    if (OP == SPMV_RESID_DRIFT && *a.drift_count == 0) return;
    for (int b = threadIdx.x; b < B; b += blockDim.x) s_act[b] = spmv_col_active(a, b) ? 1 : 0;
    double *part = red + team * B;
    if (OP != SPMV_PLAIN)
        for (int b = lane; b < B; b += 32) part[b] = 0.0;
    __syncthreads();
    const int cpl = (B + 32 * VW - 1) / (32 * VW);
    const int nteams = gridDim.x * TEAMS, gteam = blockIdx.x * TEAMS + team;
    const int per = (a.n + nteams - 1) / nteams;
    const int r0 = min(a.n, gteam * per), r1 = min(a.n, r0 + per);
    const bool use_x = OP != SPMV_RESID_INIT || a.has_x;
    const double *__restrict__ X = a.X;
    const double *__restrict__ vals = a.vals;
    const int *__restrict__ col = a.col;
    for (int k = 0; k < cpl && r0 < r1; ++k) {
        const int b = (lane + k * 32) * VW;
        const bool on = b < B;
        const unsigned bb = on ? b : 0;
        bool xp[VW];
        double al[VW];
#pragma unroll
        for (int v = 0; v < VW; ++v) {
            xp[v] = OP == SPMV_RESID_DRIFT && a.st.xpend[bb + v];
            al[v] = xp[v] ? a.st.alpha[bb + v] : 0.0;
        }
        int wb = r0, rpl = a.rp[min(r0 + lane, a.n)];  // rp[wb + lane]
        int p0 = __shfl_sync(0xffffffffu, rpl, 0), p1 = __shfl_sync(0xffffffffu, rpl, 1);
        int cj = lane < p1 - p0 ? col[p0 + lane] : r0;
        double cv = (!VB && lane < p1 - p0) ? vals[p0 + lane] : 0.0;
        for (int row = r0; row < r1; ++row) {
            const unsigned ri = (unsigned)row * B + bb;
            double own[VW];
            if (OP == SPMV_APDOT) VecT<VW>::get(*reinterpret_cast<const V *>(X + ri), own);
            else if (OP != SPMV_PLAIN) VecT<VW>::get(*reinterpret_cast<const V *>(a.Bv + ri), own);
            // the next row's bounds and first 32 entries
            int w = row + 2 - wb;
            if (w >= 32) {
                wb = row;
                rpl = a.rp[min(wb + lane, a.n)];
                w = 2;
            }
            const int q1 = __shfl_sync(0xffffffffu, rpl, w);
            const int cnt = p1 - p0, c0 = p0;
            const int ccj = cj;
            const double ccv = cv;
            if (row + 1 < r1) {
                cj = lane < q1 - p1 ? col[p1 + lane] : row + 1;
                if (!VB) cv = lane < q1 - p1 ? vals[p1 + lane] : 0.0;
            }
            p0 = p1;
            p1 = q1;
            double acc[VW];
#pragma unroll
            for (int v = 0; v < VW; ++v) acc[v] = 0.0;
            if (use_x) {
                for (int g = 0; g < cnt; g += CH) {
                    int hj = ccj;
                    double hv = ccv;
                    if (g >= 32 && (g & 31) == 0) {  // rows longer than 32 entries
                        hj = lane < cnt - g ? col[c0 + g + lane] : row;
                        hv = (!VB && lane < cnt - g) ? vals[c0 + g + lane] : 0.0;
                    }
                    double xv[CH][VW], vv[VB ? CH : 1][VW], vs[CH];
#pragma unroll
                    for (int c = 0; c < CH; ++c) {
                        const int j = __shfl_sync(0xffffffffu, hj, (g + c) & 31);
                        if (!VB) vs[c] = __shfl_sync(0xffffffffu, hv, (g + c) & 31);
                        const unsigned jo = (unsigned)j * B + bb;
                        VecT<VW>::get(*reinterpret_cast<const V *>(X + jo), xv[c]);
                        if (VB) {
                            const int e = g + c < cnt ? c0 + g + c : c0;
                            VecT<VW>::get(*reinterpret_cast<const V *>(vals + (size_t)e * B + bb), vv[c]);
                        }
                        if (OP == SPMV_RESID_DRIFT) {  // x_{k+1} = x + alpha p not yet stored (pcg.py:141)
                            double pv[VW];
                            VecT<VW>::get(*reinterpret_cast<const V *>(a.P + jo), pv);
#pragma unroll
                            for (int v = 0; v < VW; ++v)
                                if (xp[v]) xv[c][v] = __dadd_rn(xv[c][v], __dmul_rn(al[v], pv[v]));
                        }
                    }
#pragma unroll
                    for (int c = 0; c < CH; ++c) {
                        const bool use = g + c < cnt;
#pragma unroll
                        for (int v = 0; v < VW; ++v) {
                            const double s = __dadd_rn(acc[v], __dmul_rn(VB ? vv[VB ? c : 0][v] : vs[c], xv[c][v]));
                            acc[v] = use ? s : acc[v];
                        }
                    }
                }
            }
            if (on) {
#pragma unroll
                for (int v = 0; v < VW; ++v) {
                    const int bv = b + v;
                    if (!s_act[bv]) continue;
                    if (OP == SPMV_PLAIN) {
                        a.Y[ri + v] = acc[v];
                    } else if (OP == SPMV_APDOT) {
                        a.Y[ri + v] = acc[v];
                        part[bv] = __dadd_rn(part[bv], __dmul_rn(own[v], acc[v]));
                    } else {
                        const double rt = __dsub_rn(own[v], acc[v]);
                        if (OP != SPMV_RESID_FINAL) a.R[ri + v] = rt;
                        part[bv] = __dadd_rn(part[bv], __dmul_rn(rt, rt));
                    }
                }
            }
        }
    }
    if (OP == SPMV_PLAIN) return;
    spmv_reduce_tail(a, red, TEAMS);
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

// Natural <-> line order: a block moves a tile of kPermTile slots x all
// columns through shared memory, so the system-major line-order side
// ([b][slot]) and the natural RHS-minor side ([row][b]) are both read /
// written in contiguous runs.
constexpr int kPermTile = 16;

// dst[b][slot] = src[row(slot)][b] (natural RHS-minor, or shared [row] when
// src_batched == 0); padding slots get `pad`.
__global__ void __launch_bounds__(256) to_line_kernel(int nslot, int B, const int *rowof, const double *src,
                                                       int src_batched, double pad, double *dst) {
    extern __shared__ double tt[];  // [kPermTile][B + 1]
    const int ld = B + 1;
    for (int q0 = blockIdx.x * kPermTile; q0 < nslot; q0 += gridDim.x * kPermTile) {
        __syncthreads();
        for (int e = threadIdx.x; e < kPermTile * B; e += blockDim.x) {
            const int i = e / B, b = e % B;
            if (q0 + i >= nslot) continue;
            const int row = rowof[q0 + i];
            tt[i * ld + b] = row < 0 ? pad : src[src_batched ? (long long)row * B + b : row];
        }
        __syncthreads();
        for (int e = threadIdx.x; e < kPermTile * B; e += blockDim.x) {
            const int b = e / kPermTile, i = e % kPermTile;
            if (q0 + i < nslot) dst[(long long)b * nslot + q0 + i] = tt[i * ld + b];
        }
    }
}

// dst[row][b] = src[b][slot(row)]
__global__ void __launch_bounds__(256) from_line_kernel(int nslot, int B, const int *rowof, const double *src,
                                                         double *dst) {
    extern __shared__ double tt[];  // [kPermTile][B + 1]
    const int ld = B + 1;
    for (int q0 = blockIdx.x * kPermTile; q0 < nslot; q0 += gridDim.x * kPermTile) {
        __syncthreads();
        for (int e = threadIdx.x; e < kPermTile * B; e += blockDim.x) {
            const int b = e / kPermTile, i = e % kPermTile;
            if (q0 + i < nslot) tt[i * ld + b] = src[(long long)b * nslot + q0 + i];
        }
        __syncthreads();
        for (int e = threadIdx.x; e < kPermTile * B; e += blockDim.x) {
            const int i = e / B, b = e % B;
            if (q0 + i >= nslot) continue;
            const int row = rowof[q0 + i];
            if (row >= 0) dst[(long long)row * B + b] = tt[i * ld + b];
        }
    }
}

cudaError_t launch_to_line(int nslot, int B, const int *rowof, const double *src, int src_batched, double pad,
                           double *dst, cudaStream_t s) {
    const int grid = std::min((nslot + kPermTile - 1) / kPermTile, 8 * num_sms());
    note_launch();
    to_line_kernel<<<grid, 256, (size_t)kPermTile * (B + 1) * 8, s>>>(nslot, B, rowof, src, src_batched, pad, dst);
    return cudaGetLastError();
}

cudaError_t launch_from_line(int nslot, int B, const int *rowof, const double *src, double *dst, cudaStream_t s) {
    const int grid = std::min((nslot + kPermTile - 1) / kPermTile, 8 * num_sms());
    note_launch();
    from_line_kernel<<<grid, 256, (size_t)kPermTile * (B + 1) * 8, s>>>(nslot, B, rowof, src, dst);
    return cudaGetLastError();
}

// active columns and the largest iteration count (the host grows the history
// buffer from it); `finish` turns columns still ACTIVE after the pass budget
// into MAXITER so the final residual pass covers them (pcg.py:171-172)
__global__ void count_active_kernel(SolveState st, int B, long long *kmax, int finish) {
    __shared__ int s;
    __shared__ unsigned long long km;
    if (threadIdx.x == 0) s = 0, km = 0;
    __syncthreads();
    for (int b = threadIdx.x; b < B; b += blockDim.x) {
        if (st.status[b] == ST_ACTIVE) {
            if (finish) st.status[b] = ST_MAXITER;
            else atomicAdd(&s, 1);
        }
        atomicMax(&km, (unsigned long long)st.k[b]);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        *st.active_count = s;
        *kmax = (long long)km;
    }
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

// ok[b] &= vals[p] == vals[pair[p]] (sparse.py:137-147: np.array_equal on
// values, so -0.0 matches 0.0 and a NaN never matches).
__global__ void symmetric_check_kernel(long long nnz, int B, int vb, const int *pair, const double *vals,
                                       int *ok) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < nnz * B;
         q += (long long)gridDim.x * blockDim.x) {
        const long long p = q / B;
        const int b = (int)(q % B);
        const int pp = pair[p];
        const double u = vb ? vals[q] : vals[p];
        const double v = vb ? vals[(size_t)pp * B + b] : vals[pp];
        if (!(u == v)) ok[b] = 0;
    }
}

// ===========================================================================
// host launch helpers
// ===========================================================================

static std::atomic<long long> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
long long launch_count() { return g_launches.load(std::memory_order_relaxed); }

// Stream-ordered scratch (cudaMallocAsync) stays in the device pool between
// calls instead of going back to the driver at every synchronisation (the
// pool's default release threshold is 0), so repeated builds do not remap it.
void keep_pool_memory() {
    static bool done = false;
    if (done) return;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        unsigned long long keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    done = true;
}

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

static int team_lanes(int cols) {
    int tl = 1;
    while (tl < cols && tl < 32) tl <<= 1;
    return tl;
}

template <int TL, int VW>
static void spmv_launch_t(const SpmvArgs &a, int grid, size_t smem, cudaStream_t s) {
    auto kern = a.vb ? spmv_kernel<TL, VW, true> : spmv_kernel<TL, VW, false>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    note_launch();
    kern<<<grid, kSpmvThreads, smem, s>>>(a);
}

template <int VW>
static void spmv_launch_vw(int TL, const SpmvArgs &a, int grid, size_t smem, cudaStream_t s) {
    switch (TL) {
        case 1: return spmv_launch_t<1, VW>(a, grid, smem, s);
        case 2: return spmv_launch_t<2, VW>(a, grid, smem, s);
        case 4: return spmv_launch_t<4, VW>(a, grid, smem, s);
        case 8: return spmv_launch_t<8, VW>(a, grid, smem, s);
        case 16: return spmv_launch_t<16, VW>(a, grid, smem, s);
        default: return spmv_launch_t<32, VW>(a, grid, smem, s);
    }
}

template <int VW, bool VB, int OP>
static void spmv_warp_t(const SpmvArgs &a, int grid, size_t smem, cudaStream_t s) {
    auto kern = spmv_warp_kernel<VW, VB, OP>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    note_launch();
    kern<<<grid, kSpmvThreads, smem, s>>>(a);
}

template <int VW, bool VB>
static void spmv_warp_op(const SpmvArgs &a, int grid, size_t smem, cudaStream_t s) {
    switch (a.op) {
        case SPMV_PLAIN: return spmv_warp_t<VW, VB, SPMV_PLAIN>(a, grid, smem, s);
        case SPMV_APDOT: return spmv_warp_t<VW, VB, SPMV_APDOT>(a, grid, smem, s);
        case SPMV_RESID_INIT: return spmv_warp_t<VW, VB, SPMV_RESID_INIT>(a, grid, smem, s);
        case SPMV_RESID_DRIFT: return spmv_warp_t<VW, VB, SPMV_RESID_DRIFT>(a, grid, smem, s);
        default: return spmv_warp_t<VW, VB, SPMV_RESID_FINAL>(a, grid, smem, s);
    }
}

template <int VW>
static void spmv_warp_vw(const SpmvArgs &a, int grid, size_t smem, cudaStream_t s) {
    if (a.vb) spmv_warp_op<VW, true>(a, grid, smem, s);
    else spmv_warp_op<VW, false>(a, grid, smem, s);
}

// ===========================================================================
// Line-order SpMV (every operand [b][nslot], pattern.h LineSched): A in
// ELL form by slot -- ecol[e][slot] = slot of the e-th entry's column in
// the reference's row order (-1 past the row's end), evals[(b)][e][slot]
// its value. One thread owns one slot and keeps its row in registers; a
// block walks every system over its 256 slots, so matrix data is read once
// per block and every vector access of a warp is one contiguous 256-byte
// run (the row's own slot) or a gather within +-2 grid lines of it (L1).
// ===========================================================================
#ifndef NPCG_ELL_COLS
#define NPCG_ELL_COLS 32
#endif
#ifndef NPCG_ELL_NB
#define NPCG_ELL_NB 4
#endif
constexpr int kEllCols = NPCG_ELL_COLS;  // systems per block (blockIdx.y picks the group)

#ifndef NPCG_ELL_MINB
#define NPCG_ELL_MINB 2
#endif
template <int E, bool VB, int OP>
__global__ void __launch_bounds__(kSpmvThreads, NPCG_ELL_MINB) spmv_ell_kernel(SpmvArgs a) {
    constexpr int TEAMS = kSpmvThreads / 32;
    __shared__ double red[TEAMS * kSpmvThreads];  // reused by the tail's final pass
    __shared__ unsigned char s_act[kMaxBatch];
    __shared__ unsigned char s_xp[kMaxBatch];
    __shared__ double s_al[kMaxBatch];
    __shared__ unsigned char s_dr[kMaxBatch];
    const int B = a.B, ns = a.nslot, lane = threadIdx.x & 31, team = threadIdx.x >> 5;
    const int bl = blockIdx.y * kEllCols, bh = min(B, bl + kEllCols);  // this block's columns
    if (OP == SPMV_RESID_DRIFT && *a.drift_count == 0) return;
    for (int b = threadIdx.x; b < B; b += blockDim.x) {
        s_act[b] = spmv_col_active(a, b) ? 1 : 0;
        s_xp[b] = OP == SPMV_RESID_DRIFT && a.st.xpend[b];
        s_al[b] = s_xp[b] ? a.st.alpha[b] : 0.0;
        // merged drift columns: true residual from X2 (x already holds x + alpha p)
        s_dr[b] = OP == SPMV_APDOT && a.merge_drift && a.st.status[b] == ST_ACTIVE && a.st.phase[b] == PH_DRIFT;
    }
    __syncthreads();
    const int q = blockIdx.x * kSpmvThreads + threadIdx.x;
    const bool live = q < ns;
    const int qq = live ? q : 0;
    // row entries past the row's end point at the row's own slot with a zero
    // value: acc + 0 * x leaves the sum unchanged (acc starts at +0 and can
    // never become -0), so the loop needs no predicate
    unsigned cb[E];  // byte offsets of the column slots
    double v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int c = live ? a.ecol[(size_t)e * ns + q] : -1;
        cb[e] = (unsigned)(c >= 0 ? c : (live ? q : 0)) * 8u;
        v[e] = (!VB && c >= 0) ? a.evals[(size_t)e * ns + q] : 0.0;
    }
    const bool use_x = OP != SPMV_RESID_INIT || a.has_x;
    // NB systems at a time: their gathers are in flight together and their
    // dot-product trees interleave
    constexpr int NB = NPCG_ELL_NB;
    for (int b0 = bl; b0 < bh; b0 += NB) {
        // every load of the NB systems first (no branch between them), then the sums
        double xv[NB][E], own[NB];
#pragma unroll
        for (int u = 0; u < NB; ++u) {
            const int b = min(b0 + u, bh - 1);
            const size_t vb = (size_t)b * ns;
            const bool dr = OP == SPMV_APDOT && s_dr[b];
            const char *Xb = reinterpret_cast<const char *>((dr ? a.X2 : a.X) + vb);
#pragma unroll
            for (int e = 0; e < E; ++e) {
                xv[u][e] = use_x ? *reinterpret_cast<const double *>(Xb + cb[e]) : 0.0;
                if (OP == SPMV_RESID_DRIFT && s_xp[b])  // x_{k+1} = x + alpha p not yet stored (pcg.py:141)
                    xv[u][e] = __dadd_rn(xv[u][e], __dmul_rn(s_al[b], *reinterpret_cast<const double *>(
                                                                       reinterpret_cast<const char *>(a.P + vb) + cb[e])));
            }
            own[u] = (OP == SPMV_APDOT && !dr) ? a.X[vb + qq] : a.Bv[vb + qq];
        }
        double pr[NB];
#pragma unroll
        for (int u = 0; u < NB; ++u) {
            const int b = b0 + u;
            const bool on = b < bh && s_act[b] && live;
            const size_t vb = (size_t)min(b, bh - 1) * ns;
            double acc = 0.0;
#pragma unroll
            for (int e = 0; e < E; ++e) {  // sparse.py:213-219
                const double vv = VB ? a.evals[((size_t)min(b, bh - 1) * E + e) * ns + qq] : v[e];
                acc = __dadd_rn(acc, __dmul_rn(vv, xv[u][e]));
            }
            pr[u] = 0.0;
            if (OP == SPMV_APDOT && !s_dr[min(b, bh - 1)]) {
                if (on) a.Y[vb + q] = acc;
                pr[u] = on ? __dmul_rn(own[u], acc) : 0.0;  // p.Ap (pcg.py:134)
            } else {
                const double r = __dsub_rn(own[u], acc);  // r = b - A x
                if (on && OP != SPMV_RESID_FINAL) a.R[vb + q] = r;
                pr[u] = on ? __dmul_rn(r, r) : 0.0;
            }
        }
        if constexpr (NB == 4) {
            // four sums over the warp in 6 shuffles instead of 20: the first two butterfly
            // steps also halve the values a lane carries (lanes 0-7 end with system 0's
            // total, 8-15 system 1's, 16-23 system 2's, 24-31 system 3's); fixed order
            const bool h16 = lane & 16, h8 = lane & 8;
            double k0 = h16 ? pr[2] : pr[0], k1 = h16 ? pr[3] : pr[1];
            const double s0 = h16 ? pr[0] : pr[2], s1 = h16 ? pr[1] : pr[3];
            k0 = __dadd_rn(k0, __shfl_xor_sync(0xffffffffu, s0, 16));
            k1 = __dadd_rn(k1, __shfl_xor_sync(0xffffffffu, s1, 16));
            double kk = h8 ? k1 : k0;
            const double ss = h8 ? k0 : k1;
            kk = __dadd_rn(kk, __shfl_xor_sync(0xffffffffu, ss, 8));
#pragma unroll
            for (int off = 4; off > 0; off >>= 1) kk = __dadd_rn(kk, __shfl_xor_sync(0xffffffffu, kk, off));
            const int u = lane >> 3;
            if ((lane & 7) == 0 && b0 + u < bh) red[team * kEllCols + b0 + u - bl] = kk;
        } else {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1)
#pragma unroll
                for (int u = 0; u < NB; ++u) pr[u] = __dadd_rn(pr[u], __shfl_down_sync(0xffffffffu, pr[u], off));
            if (lane == 0)
#pragma unroll
                for (int u = 0; u < NB; ++u)
                    if (b0 + u < bh) red[team * kEllCols + b0 + u - bl] = pr[u];
        }
    }
    spmv_reduce_tail(a, red, TEAMS, bl, bh, kEllCols);
}

template <int E, bool VB>
static void spmv_ell_op(const SpmvArgs &a, dim3 grid, cudaStream_t s) {
    note_launch();
    switch (a.op) {
        case SPMV_APDOT: spmv_ell_kernel<E, VB, SPMV_APDOT><<<grid, kSpmvThreads, 0, s>>>(a); break;
        case SPMV_RESID_INIT: spmv_ell_kernel<E, VB, SPMV_RESID_INIT><<<grid, kSpmvThreads, 0, s>>>(a); break;
        case SPMV_RESID_DRIFT: spmv_ell_kernel<E, VB, SPMV_RESID_DRIFT><<<grid, kSpmvThreads, 0, s>>>(a); break;
        default: spmv_ell_kernel<E, VB, SPMV_RESID_FINAL><<<grid, kSpmvThreads, 0, s>>>(a); break;
    }
}

template <int E>
static void spmv_ell_e(const SpmvArgs &a, dim3 grid, cudaStream_t s) {
    if (a.vb) spmv_ell_op<E, true>(a, grid, s);
    else spmv_ell_op<E, false>(a, grid, s);
}

static cudaError_t launch_spmv_ell(const SpmvArgs &a, cudaStream_t s) {
    if (a.op == SPMV_PLAIN || a.nslot <= 0) return cudaErrorInvalidValue;
    const dim3 grid((a.nslot + kSpmvThreads - 1) / kSpmvThreads, (a.B + kEllCols - 1) / kEllCols);
    if ((size_t)grid.x * a.B > a.partial_cap) return cudaErrorInvalidValue;
    switch (a.ell_width) {
        case 4: spmv_ell_e<4>(a, grid, s); break;
        case 7: spmv_ell_e<7>(a, grid, s); break;
        case 8: spmv_ell_e<8>(a, grid, s); break;
        case 12: spmv_ell_e<12>(a, grid, s); break;
        case 16: spmv_ell_e<16>(a, grid, s); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// p = z + beta p | p = z ; x += alpha p, every vector in line order (pcg.py:129, 141, 170);
// x == nullptr: the x update is xupd_ell_kernel's
__global__ void __launch_bounds__(256) pupd_ell_kernel(int nslot, const double *z, double *p, double *x,
                                                        SolveState st) {
    const int b = blockIdx.y;
    int f = st.pflag[b];
    if (!x) f &= ~PF_X;
    if (f == PF_NONE) return;
    const double al = st.alpha[b], be = st.beta[b];
    const size_t vb = (size_t)b * nslot;
    const double2 *z2 = reinterpret_cast<const double2 *>(z + vb);
    double2 *p2 = reinterpret_cast<double2 *>(p + vb), *x2 = reinterpret_cast<double2 *>(x + vb);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nslot / 2; i += gridDim.x * blockDim.x) {
        double2 pq = p2[i];
        if (f & PF_X) {
            double2 xq = x2[i];
            xq.x = __dadd_rn(xq.x, __dmul_rn(al, pq.x));
            xq.y = __dadd_rn(xq.y, __dmul_rn(al, pq.y));
            x2[i] = xq;
        }
        if (f & (PF_UPDATE | PF_COPY)) {
            const double2 zq = z2[i];
            if (f & PF_UPDATE) {
                pq.x = __dadd_rn(zq.x, __dmul_rn(be, pq.x));
                pq.y = __dadd_rn(zq.y, __dmul_rn(be, pq.y));
            } else {
                pq = zq;
            }
            p2[i] = pq;
        }
    }
}

cudaError_t launch_pupd_ell(int nslot, int B, const double *z, double *p, double *x, const SolveState &st,
                            cudaStream_t s) {
    const int per = (nslot / 2 + 255) / 256;
    const int gx = std::max(1, std::min(per, (4 * num_sms() + B - 1) / B));
    note_launch();
    pupd_ell_kernel<<<dim3(gx, B), 256, 0, s>>>(nslot, z, p, x, st);
    return cudaGetLastError();
}

// x += alpha p (pcg.py:141) for the columns whose alpha this pass's SpMV formed (st.xgo[b] ==
// st.epoch): needs p_k and alpha only, so it runs beside the P^{-1} launch on a side stream
__global__ void __launch_bounds__(256) xupd_ell_kernel(int nslot, const double *p, double *x, SolveState st) {
    const int b = blockIdx.y;
    if (st.xgo[b] != st.epoch) return;
    const double al = st.alpha[b];
    const size_t vb = (size_t)b * nslot;
    const double2 *p2 = reinterpret_cast<const double2 *>(p + vb);
    double2 *x2 = reinterpret_cast<double2 *>(x + vb);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nslot / 2; i += gridDim.x * blockDim.x) {
        const double2 pq = p2[i];
        double2 xq = x2[i];
        xq.x = __dadd_rn(xq.x, __dmul_rn(al, pq.x));
        xq.y = __dadd_rn(xq.y, __dmul_rn(al, pq.y));
        x2[i] = xq;
    }
}

cudaError_t launch_xupd_ell(int nslot, int B, const double *p, double *x, const SolveState &st, cudaStream_t s) {
    const int per = (nslot / 2 + 255) / 256;
    const int gx = std::max(1, std::min(per, (2 * num_sms() + B - 1) / B));
    note_launch();
    xupd_ell_kernel<<<dim3(gx, B), 256, 0, s>>>(nslot, p, x, st);
    return cudaGetLastError();
}

// packed[b][e] = S[perm[e] * ps + b * bs]  (0 where perm < 0)
__global__ void gather_pack_kernel(long long per, int B, int sb, long long ps, long long bs, const int *perm,
                                   const double *S, double *packed) {
    const long long total = per * (sb ? B : 1);
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
         q += (long long)gridDim.x * blockDim.x) {
        const long long b = q / per, e = q % per;
        const int p = perm[e];
        packed[q] = p < 0 ? 0.0 : S[(long long)p * ps + b * bs];
    }
}

void launch_gather_pack(long long per, int B, int sb, long long ps, long long bs, const int *perm, const double *S,
                        double *packed, cudaStream_t s) {
    const long long total = per * (sb ? B : 1);
    note_launch();
    gather_pack_kernel<<<(int)std::min<long long>((total + 255) / 256, 16384), 256, 0, s>>>(per, B, sb, ps, bs, perm,
                                                                                             S, packed);
}

// dst[q * B + b] = src[sel[q] * B + b]: rows of a column-minor (count, B) array
__global__ void gather_rows_kernel(long long count, int B, const int *sel, const double *src, double *dst) {
    const long long total = count * B;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
        const long long q = t / B;
        dst[t] = src[(long long)sel[q] * B + (t - q * B)];
    }
}

void launch_gather_rows(long long count, int B, const int *sel, const double *src, double *dst, cudaStream_t s) {
    const long long total = count * B;
    if (total <= 0) return;
    note_launch();
    gather_rows_kernel<<<(int)std::min<long long>((total + 255) / 256, 16384), 256, 0, s>>>(count, B, sel, src, dst);
}

cudaError_t launch_spmv(const SpmvArgs &a, cudaStream_t s) {
    if (a.ecol) return launch_spmv_ell(a, s);
    // 16-byte column pairs when every row of every operand stays 16-byte aligned
    auto al16 = [](const void *p) { return p == nullptr || ((uintptr_t)p & 15) == 0; };
    const bool even16 = a.B % 2 == 0 && al16(a.X) && al16(a.Y) && al16(a.Bv) && al16(a.R) && al16(a.P) &&
                        (!a.vb || al16(a.vals));
    // four columns per lane (one pass over the rows) for wide shared-matrix
    // batches: twice the gathers in flight per row (NPCG_SPMV_VW4=0 disables)
    static const bool vw4_on = [] {
        const char *env = std::getenv("NPCG_SPMV_VW4");
        return !env || std::atoi(env) != 0;
    }();
    const int VW = (even16 && vw4_on && a.B % 4 == 0 && a.B >= 128 && !a.vb && a.op != SPMV_RESID_DRIFT) ? 4 : even16 ? 2 : 1;
    const int TL = team_lanes((a.B + VW - 1) / VW);
    const int teams = kSpmvThreads / TL;
    long long need = (a.n + teams - 1) / teams;
    int grid;
    if (a.op == SPMV_PLAIN) grid = (int)std::min<long long>(std::max<long long>(need, 1), 65535);
    else grid = (int)std::min<long long>(std::max<long long>(need, 1), (long long)kReduceBlocksPerSm * num_sms());
    size_t smem = a.op == SPMV_PLAIN ? 0 : (size_t)teams * a.B * sizeof(double);
    smem = std::max(smem, (size_t)kSpmvThreads * sizeof(double));
    if (VW == 4 && (long long)a.n * a.B < (1ll << 31)) {
        switch (a.op) {  // the drift op keeps two columns per lane (register pressure)
            case SPMV_PLAIN: spmv_warp_t<4, false, SPMV_PLAIN>(a, grid, smem, s); break;
            case SPMV_APDOT: spmv_warp_t<4, false, SPMV_APDOT>(a, grid, smem, s); break;
            case SPMV_RESID_INIT: spmv_warp_t<4, false, SPMV_RESID_INIT>(a, grid, smem, s); break;
            default: spmv_warp_t<4, false, SPMV_RESID_FINAL>(a, grid, smem, s); break;
        }
    } else if (TL == 32 && (long long)a.n * a.B < (1ll << 31)) {
        if (VW == 2) spmv_warp_vw<2>(a, grid, smem, s);
        else spmv_warp_vw<1>(a, grid, smem, s);
    } else if (VW == 2) {
        spmv_launch_vw<2>(TL, a, grid, smem, s);
    } else {
        spmv_launch_vw<1>(TL, a, grid, smem, s);
    }
    return cudaGetLastError();
}

}  // namespace npcg
