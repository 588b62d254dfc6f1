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

int level_sync_grid(int B) {
    if (B < 1 || B > 256) return 0;
    const int T = B * std::max(1, 256 / B);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, level_sync_kernel<false, true>, T, (size_t)T * 8);
    int cap = 8;  // blocks per SM (occupancy-limited): measured 68 / 95 / 111 systems/s at 1 / 2 / 4, config 4
    if (const char *env = std::getenv("NPCG_LEVELSYNC_OCC")) cap = std::max(1, std::atoi(env));
    occ = std::max(1, std::min(occ, cap));
    return occ * num_sms();
}

cudaError_t launch_level_sync(const LevelSyncArgs &a, cudaStream_t s) {
    if (a.B < 1 || a.B > 256 || !a.bar) return cudaErrorInvalidValue;
    const int T = a.B * std::max(1, 256 / a.B);
    const int grid = a.grid > 0 ? a.grid : level_sync_grid(a.B);
    void *args[] = {const_cast<LevelSyncArgs *>(&a)};
    const bool pcg = a.mode == TRSV_PCG;
    const void *fn = a.upper ? (pcg ? (const void *)level_sync_kernel<true, true> : (const void *)level_sync_kernel<true, false>)
                             : (pcg ? (const void *)level_sync_kernel<false, true> : (const void *)level_sync_kernel<false, false>);
    note_launch();
    // cooperative: every block resident at once (the grid barrier relies on it)
    return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(T), args, (size_t)T * 8, s);
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
