// trsv_level.cu -- level-synchronous triangular solves for batches on
// patterns without a line schedule (3-D Kuhn meshes: 187 levels at config 4,
// 385 at config 5; sparse.py:222-239, 265-275).
//
// One cooperative launch per direction walks the global level sets
// (pattern.h LevelDir) with a grid-wide barrier between levels. A level's
// rows are independent, and every one of them is solved for the whole
// batch at once: thread (row lane, b) owns column b of its rows, so a
// warp's loads of a dependency (one row, 32 adjacent columns of the
// RHS-minor vectors) are one coalesced 256-byte access and the factor
// value is a broadcast (shared factor) or coalesced too (per-system
// factors stored [entry][B]). Where the chunked level kernel (trsv.cu)
// runs one column per unit in ~20 latency-bound waves, a level here is one
// pass over rows x batch for the whole GPU.
//
// Sums keep the reference's order with unfused fp64 operations (bitwise the
// reference); the backward solve divides y / D exactly as it reads its own
// row. PCG mode fuses r -= alpha Ap with |r|^2 into the forward solve and
// r.z into the backward one (fixed-order reductions), and runs the per-
// column epilogues (common.cuh) at the end.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "trsv.cuh"

namespace npcg {

namespace {

// sense-free grid barrier: count arrivals, the last one advances the generation
__device__ __forceinline__ void grid_barrier(unsigned *count, unsigned *gen, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned *vg = gen;
        const unsigned g = *vg;
        __threadfence();
        if (atomicAdd(count, 1u) == nblocks - 1) {
            *count = 0;
            __threadfence();
            atomicAdd(gen, 1u);
        } else {
            while (*vg == g) __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
}

}  // namespace

template <bool UPPER, bool PCG>
__global__ void __launch_bounds__(256) level_sync_kernel(LevelSyncArgs a) {
    extern __shared__ double red[];  // [blockDim.x]
    const int B = a.B, T = blockDim.x, rpb = T / B;
    const int b = threadIdx.x % B, lane = blockIdx.x * rpb + threadIdx.x / B;
    const int lanes = gridDim.x * rpb;
    const bool in_use = threadIdx.x < rpb * B;
    // what column b needs (pcg.py:128-171 phases, common.cuh)
    int op = TOP_SOLVE;
    if (PCG) {
        const SolveState &st = a.st;
        if (st.status[b] != ST_ACTIVE) op = TOP_SKIP;
        else {
            const int ph = st.phase[b];
            op = !UPPER ? (ph == PH_ITER ? TOP_UPDATE : (ph == PH_INIT ? TOP_SOLVE : TOP_SKIP))
                        : ((ph == PH_ITER || ph == PH_INIT) ? TOP_SOLVE : TOP_SKIP);
        }
    }
    const double alpha = (PCG && op == TOP_UPDATE) ? a.st.alpha[b] : 0.0;
    const size_t sbs = a.s_batched ? (size_t)B : 0;
    double part = 0.0;
    for (int L = 0; L < a.nlev; ++L) {
        if (in_use && op != TOP_SKIP) {
            const int k1 = a.lvl_ptr[L + 1];
            for (int k = a.lvl_ptr[L] + lane; k < k1; k += lanes) {
                const int i = a.rows[k];
                const size_t ib = (size_t)i * B + b;
                double acc;
                if (UPPER) {
                    acc = __ddiv_rn(a.in[ib], a.D[a.d_batched ? ib : (size_t)i]);  // y / D (sparse.py:273)
                } else {
                    acc = a.in[ib];
                    if (PCG && op == TOP_UPDATE) {  // r_{k+1} = r_k - alpha A p (pcg.py:142-143)
                        acc = __dsub_rn(acc, __dmul_rn(alpha, a.AP[ib]));
                        a.R[ib] = acc;
                        part = __dadd_rn(part, __dmul_rn(acc, acc));
                    }
                }
                // dependencies in groups of 8: every load of a group in flight before
                // the group's terms are subtracted in the reference's order
                const int e0 = a.eptr[k], e1 = a.eptr[k + 1];
                for (int e = e0; e < e1; e += 8) {
                    double f[8], y[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int ee = e + u < e1 ? e + u : e;
                        f[u] = a.S[(size_t)ee * (sbs ? sbs : 1) + (sbs ? b : 0)];
                        y[u] = a.out[(size_t)a.ecol[ee] * B + b];
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        if (e + u < e1) acc = __dsub_rn(acc, __dmul_rn(f[u], y[u]));
                }
                a.out[ib] = acc;
                if (UPPER && PCG) part = __dadd_rn(part, __dmul_rn(a.R[ib], acc));  // r.z (pcg.py:167)
            }
        }
        grid_barrier(a.bar, a.bar + 1, gridDim.x);
    }
    if (!PCG) return;
    // fixed-order reductions: the block's threads of column b, then the blocks
    red[threadIdx.x] = part;
    __syncthreads();
    if (threadIdx.x < B) {
        double s = 0.0;
        for (int r = 0; r < rpb; ++r) s = __dadd_rn(s, red[r * B + threadIdx.x]);
        a.partial[(size_t)blockIdx.x * B + threadIdx.x] = s;
    }
    grid_barrier(a.bar, a.bar + 1, gridDim.x);
    if (blockIdx.x == 0)
        for (int c = threadIdx.x; c < B; c += T) {
            double s = 0.0;
            for (int g = 0; g < (int)gridDim.x; ++g) s = __dadd_rn(s, __ldcg(&a.partial[(size_t)g * B + c]));
            if (UPPER) bwd_epilogue(a.st, c, s);
            else fwd_epilogue(a.st, c, s, a.drift_count);
        }
}

__device__ __forceinline__ unsigned ld_flag(const unsigned *p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_flag(unsigned *p, unsigned v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Dependency-flag variant: no barrier between levels. The level-ordered row
// list is dealt round-robin to lanes (row groups); a lane solves its rows in
// list order, and before reading a dependency's y it waits for that row's
// flag (same column group) to reach this launch's epoch. A row publishes its
// flag after its stores are fenced. Level order is topological, so the
// smallest unfinished position always has its dependencies done: with every
// block resident (cooperative launch) the walk cannot deadlock, and a row
// starts as soon as its own dependencies are final instead of when the whole
// previous level is. Dependency values are read from L2 (ld.cg) after the
// flag is observed: loads issue in order behind the flag test.
// WARPF: one flag per (row, 32-column warp) set by lane 0 after __syncwarp
// (B % 32 == 0); otherwise one flag per (row, column).
template <bool UPPER, bool PCG, bool WARPF>
__global__ void __launch_bounds__(256) level_flag_kernel(LevelSyncArgs a) {
    extern __shared__ double red[];  // [blockDim.x]
    const int B = a.B, T = blockDim.x, rpb = T / B;
    const int b = threadIdx.x % B, lane = blockIdx.x * rpb + threadIdx.x / B;
    const int lanes = gridDim.x * rpb;
    const bool in_use = threadIdx.x < rpb * B;
    const int nf = WARPF ? B / 32 : B, fg = WARPF ? b / 32 : b;
    const unsigned epoch = a.epoch;
    int op = TOP_SOLVE;
    if (PCG) {
        const SolveState &st = a.st;
        if (st.status[b] != ST_ACTIVE) op = TOP_SKIP;
        else {
            const int ph = st.phase[b];
            op = !UPPER ? (ph == PH_ITER ? TOP_UPDATE : (ph == PH_INIT ? TOP_SOLVE : TOP_SKIP))
                        : ((ph == PH_ITER || ph == PH_INIT) ? TOP_SOLVE : TOP_SKIP);
        }
    }
    const double alpha = (PCG && op == TOP_UPDATE) ? a.st.alpha[b] : 0.0;
    const size_t sbs = a.s_batched ? (size_t)B : 0;
    double part = 0.0;
    const int nrows = a.lvl_ptr[a.nlev];
    if (in_use)
        for (int k = lane; k < nrows; k += lanes) {
            const int i = a.rows[k];
            if (op != TOP_SKIP) {
                const size_t ib = (size_t)i * B + b;
                double acc;
                if (UPPER) {
                    acc = __ddiv_rn(a.in[ib], a.D[a.d_batched ? ib : (size_t)i]);  // y / D (sparse.py:273)
                } else {
                    acc = a.in[ib];
                    if (PCG && op == TOP_UPDATE) {  // r_{k+1} = r_k - alpha A p (pcg.py:142-143)
                        acc = __dsub_rn(acc, __dmul_rn(alpha, a.AP[ib]));
                        a.R[ib] = acc;
                        part = __dadd_rn(part, __dmul_rn(acc, acc));
                    }
                }
                const int e0 = a.eptr[k], e1 = a.eptr[k + 1];
                for (int e = e0; e < e1; e += 8) {
                    int c[8];
                    double f[8], y[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int ee = e + u < e1 ? e + u : e;
                        c[u] = a.ecol[ee];
                        f[u] = a.S[(size_t)ee * (sbs ? sbs : 1) + (sbs ? b : 0)];
                    }
                    // poll the group's flags together: all loads in flight at once
                    unsigned need = e1 - e >= 8 ? 0xffu : (1u << (e1 - e)) - 1u;
                    for (;;) {
                        unsigned v[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) v[u] = (need >> u) & 1u ? ld_flag(&a.flags[(size_t)c[u] * nf + fg]) : epoch;
#pragma unroll
                        for (int u = 0; u < 8; ++u)
                            if (v[u] >= epoch) need &= ~(1u << u);
                        if (!need) break;
                        __nanosleep(a.sleep_ns);
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) y[u] = __ldcg(&a.out[(size_t)c[u] * B + b]);
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        if (e + u < e1) acc = __dsub_rn(acc, __dmul_rn(f[u], y[u]));
                }
                a.out[ib] = acc;
                if (UPPER && PCG) part = __dadd_rn(part, __dmul_rn(a.R[ib], acc));  // r.z (pcg.py:167)
            }
            __threadfence();
            if (WARPF) {
                __syncwarp();
                if ((threadIdx.x & 31) == 0) st_flag(&a.flags[(size_t)i * nf + fg], epoch);
            } else {
                st_flag(&a.flags[(size_t)i * nf + fg], epoch);
            }
        }
    if (!PCG) return;
    red[threadIdx.x] = part;
    __syncthreads();
    if (threadIdx.x < B) {
        double s = 0.0;
        for (int r = 0; r < rpb; ++r) s = __dadd_rn(s, red[r * B + threadIdx.x]);
        a.partial[(size_t)blockIdx.x * B + threadIdx.x] = s;
    }
    grid_barrier(a.bar, a.bar + 1, gridDim.x);
    if (blockIdx.x == 0)
        for (int c = threadIdx.x; c < B; c += T) {
            double s = 0.0;
            for (int g = 0; g < (int)gridDim.x; ++g) s = __dadd_rn(s, __ldcg(&a.partial[(size_t)g * B + c]));
            if (UPPER) bwd_epilogue(a.st, c, s);
            else fwd_epilogue(a.st, c, s, a.drift_count);
        }
}

// Warp-per-row variant of the flag walk (B a multiple of 32): a warp owns
// one row for 32 x VW adjacent columns (VW per lane, vector loads), so a
// row's index data are warp-uniform and loaded once per warp -- lane u
// fetches dependency u's column index and factor value and polls its flag,
// one vote decides, then every lane loads the VW-column slices of the ready
// dependencies (one coalesced 256 x VW-byte access each). WPR warps cover a
// row when B > 32 x VW; one flag word per (row, warp group).
template <int VW>
struct VecD;
template <>
struct VecD<1> {
    static __device__ __forceinline__ void ld(double *d, const double *p) { d[0] = __ldcg(p); }
    static __device__ __forceinline__ void ld_nc(double *d, const double *p) { d[0] = *p; }
    static __device__ __forceinline__ void st(double *p, const double *d) { *p = d[0]; }
};
template <>
struct VecD<2> {
    static __device__ __forceinline__ void ld(double *d, const double *p) {
        const double2 v = __ldcg(reinterpret_cast<const double2 *>(p));
        d[0] = v.x, d[1] = v.y;
    }
    static __device__ __forceinline__ void ld_nc(double *d, const double *p) {
        const double2 v = *reinterpret_cast<const double2 *>(p);
        d[0] = v.x, d[1] = v.y;
    }
    static __device__ __forceinline__ void st(double *p, const double *d) {
        *reinterpret_cast<double2 *>(p) = make_double2(d[0], d[1]);
    }
};
template <>
struct VecD<4> {
    static __device__ __forceinline__ void ld(double *d, const double *p) {
        VecD<2>::ld(d, p);
        VecD<2>::ld(d + 2, p + 2);
    }
    static __device__ __forceinline__ void ld_nc(double *d, const double *p) {
        VecD<2>::ld_nc(d, p);
        VecD<2>::ld_nc(d + 2, p + 2);
    }
    static __device__ __forceinline__ void st(double *p, const double *d) {
        VecD<2>::st(p, d);
        VecD<2>::st(p + 2, d + 2);
    }
};

template <bool UPPER, bool PCG, int VW>
__global__ void __launch_bounds__(256, 2) level_warp_kernel(LevelSyncArgs a) {
    extern __shared__ double red[];  // [8 warps][32 * VW]
    const int B = a.B, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int wpr = B / (32 * VW), rpb = 8 / wpr;
    const int g = w % wpr, rl = w / wpr;
    const int col = g * 32 * VW + lane * VW;  // first of this lane's VW columns
    const int my = blockIdx.x * rpb + rl, lanes = gridDim.x * rpb;
    const unsigned epoch = a.epoch;
    const bool sb = a.s_batched != 0;
    int op[VW];
    double alpha[VW], part[VW];
#pragma unroll
    for (int v = 0; v < VW; ++v) {
        op[v] = TOP_SOLVE;
        alpha[v] = 0.0;
        part[v] = 0.0;
        if (PCG) {
            const int b = col + v;
            if (a.st.status[b] != ST_ACTIVE) op[v] = TOP_SKIP;
            else {
                const int ph = a.st.phase[b];
                op[v] = !UPPER ? (ph == PH_ITER ? TOP_UPDATE : (ph == PH_INIT ? TOP_SOLVE : TOP_SKIP))
                               : ((ph == PH_ITER || ph == PH_INIT) ? TOP_SOLVE : TOP_SKIP);
            }
            if (op[v] == TOP_UPDATE) alpha[v] = a.st.alpha[b];
        }
    }
    bool any = false, all = true;
#pragma unroll
    for (int v = 0; v < VW; ++v) {
        any |= op[v] != TOP_SKIP;
        all &= op[v] != TOP_SKIP;
    }
    const bool warp_any = __any_sync(~0u, any);
    const int nrows = a.lvl_ptr[a.nlev];
    for (int k = my; k < nrows; k += lanes) {
        const int i = a.rows[k];
        if (warp_any) {
            const size_t ib = (size_t)i * B + col;
            double acc[VW];
            VecD<VW>::ld_nc(acc, a.in + ib);
            if (UPPER) {  // y / D (sparse.py:273)
                double d[VW];
                if (a.d_batched) VecD<VW>::ld_nc(d, a.D + ib);
                else {
#pragma unroll
                    for (int v = 0; v < VW; ++v) d[v] = a.D[i];
                }
#pragma unroll
                for (int v = 0; v < VW; ++v) acc[v] = __ddiv_rn(acc[v], d[v]);
            } else if (PCG) {  // r_{k+1} = r_k - alpha A p (pcg.py:142-143)
                double ap[VW];
                VecD<VW>::ld_nc(ap, a.AP + ib);
#pragma unroll
                for (int v = 0; v < VW; ++v)
                    if (op[v] == TOP_UPDATE) {
                        acc[v] = __dsub_rn(acc[v], __dmul_rn(alpha[v], ap[v]));
                        a.R[ib + v] = acc[v];
                        part[v] = __dadd_rn(part[v], __dmul_rn(acc[v], acc[v]));
                    }
            }
            const int e0 = a.eptr[k], e1 = a.eptr[k + 1];
            for (int e = e0; e < e1; e += 8) {
                const int m = min(8, e1 - e);
                const int cl = lane < m ? a.ecol[e + lane] : 0;
                const double fl = (!sb && lane < m) ? a.S[e + lane] : 0.0;
                // lane u polls dependency u; one vote for the group
                for (;;) {
                    const bool ok = lane >= m || ld_flag(&a.flags[(size_t)cl * wpr + g]) >= epoch;
                    if (__all_sync(~0u, ok)) break;
                    __nanosleep(a.sleep_ns);
                }
                double y[8][VW];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int c = __shfl_sync(~0u, cl, u);
                    if (u < m) VecD<VW>::ld(y[u], a.out + (size_t)c * B + col);
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    if (u < m) {
                        double f[VW];
                        if (sb) VecD<VW>::ld_nc(f, a.S + (size_t)(e + u) * B + col);
                        else {
                            const double fu = __shfl_sync(~0u, fl, u);
#pragma unroll
                            for (int v = 0; v < VW; ++v) f[v] = fu;
                        }
#pragma unroll
                        for (int v = 0; v < VW; ++v) acc[v] = __dsub_rn(acc[v], __dmul_rn(f[v], y[u][v]));
                    }
                }
            }
            if (all) VecD<VW>::st(a.out + ib, acc);
            else {
#pragma unroll
                for (int v = 0; v < VW; ++v)
                    if (op[v] != TOP_SKIP) a.out[ib + v] = acc[v];
            }
            if (UPPER && PCG) {  // r.z (pcg.py:167)
                double r[VW];
                VecD<VW>::ld_nc(r, a.R + ib);
#pragma unroll
                for (int v = 0; v < VW; ++v)
                    if (op[v] != TOP_SKIP) part[v] = __dadd_rn(part[v], __dmul_rn(r[v], acc[v]));
            }
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) st_flag(&a.flags[(size_t)i * wpr + g], epoch);
    }
    if (!PCG) return;
    // fixed-order reductions: the block's row lanes of each column, then the blocks
#pragma unroll
    for (int v = 0; v < VW; ++v) red[rl * B + col + v] = part[v];
    __syncthreads();
    for (int c = threadIdx.x; c < B; c += blockDim.x) {
        double s = 0.0;
        for (int r = 0; r < rpb; ++r) s = __dadd_rn(s, red[r * B + c]);
        a.partial[(size_t)blockIdx.x * B + c] = s;
    }
    grid_barrier(a.bar, a.bar + 1, gridDim.x);
    if (blockIdx.x == 0)
        for (int c = threadIdx.x; c < B; c += blockDim.x) {
            double s = 0.0;
            for (int q = 0; q < (int)gridDim.x; ++q) s = __dadd_rn(s, __ldcg(&a.partial[(size_t)q * B + c]));
            if (UPPER) bwd_epilogue(a.st, c, s);
            else fwd_epilogue(a.st, c, s, a.drift_count);
        }
}

// warp-per-row shape for B, or 0: VW columns per lane, B / (32 VW) warps per row dividing 8
static int level_warp_vw(int B) {
    if (B < 32 || B % 32) return 0;
    const int vw = B >= 128 ? 4 : B / 32;
    const int wpr = B / (32 * vw);
    return (vw == 1 || vw == 2 || vw == 4) && B % (32 * vw) == 0 && 8 % wpr == 0 ? vw : 0;
}

template <bool UPPER, bool PCG>
static const void *level_warp_fn(int B) {
    switch (level_warp_vw(B)) {
        case 1: return (const void *)level_warp_kernel<UPPER, PCG, 1>;
        case 2: return (const void *)level_warp_kernel<UPPER, PCG, 2>;
        case 4: return (const void *)level_warp_kernel<UPPER, PCG, 4>;
    }
    return nullptr;
}


namespace {

struct LevelShape {
    const void *fn = nullptr;
    int T = 0, rows_per_block = 0;
    size_t smem = 0;
};

// kernel variant and block shape: the barrier walk, or the flag walk (warp per
// row when B allows, else thread per column)
LevelShape level_shape(int B, bool upper, bool pcg, bool flags) {
    LevelShape sh;
    if (flags && level_warp_vw(B)) {
        const int vw = level_warp_vw(B);
        sh.fn = upper ? (pcg ? level_warp_fn<true, true>(B) : level_warp_fn<true, false>(B))
                      : (pcg ? level_warp_fn<false, true>(B) : level_warp_fn<false, false>(B));
        sh.T = 256;
        sh.rows_per_block = 8 / (B / (32 * vw));
        sh.smem = (size_t)256 * vw * 8;
        return sh;
    }
    sh.T = B * std::max(1, 256 / B);
    sh.rows_per_block = sh.T / B;
    sh.smem = (size_t)sh.T * 8;
    if (flags) {
        const bool wf = B % 32 == 0;
        sh.fn = upper ? (pcg ? (wf ? (const void *)level_flag_kernel<true, true, true> : (const void *)level_flag_kernel<true, true, false>)
                             : (wf ? (const void *)level_flag_kernel<true, false, true> : (const void *)level_flag_kernel<true, false, false>))
                      : (pcg ? (wf ? (const void *)level_flag_kernel<false, true, true> : (const void *)level_flag_kernel<false, true, false>)
                             : (wf ? (const void *)level_flag_kernel<false, false, true> : (const void *)level_flag_kernel<false, false, false>));
    } else {
        sh.fn = upper ? (pcg ? (const void *)level_sync_kernel<true, true> : (const void *)level_sync_kernel<true, false>)
                      : (pcg ? (const void *)level_sync_kernel<false, true> : (const void *)level_sync_kernel<false, false>);
    }
    return sh;
}

// co-resident blocks of one variant (capped per SM: NPCG_LEVELSYNC_OCC)
int coop_grid(const LevelShape &sh) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sh.fn, sh.T, sh.smem);
    int cap = 8;  // barrier walk, config 4: 68 / 95 / 111 systems/s at 1 / 2 / 4 blocks per SM
    if (const char *env = std::getenv("NPCG_LEVELSYNC_OCC")) cap = std::max(1, std::atoi(env));
    return std::max(1, std::min(occ, cap)) * num_sms();
}

}  // namespace

int level_sync_grid(int B) {  // the largest grid any variant launches (partial-sum rows)
    if (B < 1 || B > 256) return 0;
    int grid = 0;
    for (int f = 0; f < 2; ++f)
        for (int u = 0; u < 2; ++u)
            for (int p = 0; p < 2; ++p) grid = std::max(grid, coop_grid(level_shape(B, u, p, f)));
    return grid;
}

cudaError_t launch_level_sync(const LevelSyncArgs &a, cudaStream_t s) {
    if (a.B < 1 || a.B > 256 || !a.bar) return cudaErrorInvalidValue;
    const LevelShape sh = level_shape(a.B, a.upper != 0, a.mode == TRSV_PCG, a.flags != nullptr);
    LevelSyncArgs c = a;
    int grid = coop_grid(sh);
    if (a.grid > 0) grid = std::min(grid, a.grid);
    else if (a.flags) {
        // flag mode: lanes for `width` x the widest level, not more -- idle lanes
        // only poll (NPCG_LEVELFLAG_WIDTH, 0 = the full co-resident grid)
        double width = 4.0;
        if (const char *env = std::getenv("NPCG_LEVELFLAG_WIDTH")) width = std::atof(env);
        if (width > 0) {
            const int want = (int)std::ceil(width * std::max(1, a.max_rows) / sh.rows_per_block);
            grid = std::max(std::min(grid, num_sms()), std::min(grid, want));
        }
    }
    if (const char *env = std::getenv("NPCG_LEVELFLAG_SLEEP")) c.sleep_ns = std::max(0, std::atoi(env));
    void *args[] = {&c};
    note_launch();
    // cooperative: every block resident at once (the grid barrier and the flag walk rely on it)
    return cudaLaunchCooperativeKernel(sh.fn, dim3(grid), dim3(sh.T), args, sh.smem, s);
}

__global__ void level_factor_pack_kernel(long long entries, int B, int sb, const int *perm, const double *S,
                                         double *packed) {
    const long long total = entries * (sb ? B : 1);
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total; q += (long long)gridDim.x * blockDim.x) {
        if (sb) {
            const long long e = q / B;
            const int b = (int)(q % B);
            packed[q] = S[(size_t)perm[e] * B + b];
        } else {
            packed[q] = S[perm[q]];
        }
    }
}

void launch_level_factor_pack(long long entries, int B, int sb, const int *perm, const double *S, double *packed,
                              cudaStream_t s) {
    const long long total = entries * (sb ? B : 1);
    if (total <= 0) return;
    note_launch();
    level_factor_pack_kernel<<<(int)std::min<long long>((total + 255) / 256, 16384), 256, 0, s>>>(entries, B, sb, perm,
                                                                                                 S, packed);
}

}  // namespace npcg
