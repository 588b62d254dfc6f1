// trsv_line.cu -- line-wavefront triangular solves for patterns whose rows
// form at most 1024 "lines" (runs of rows each depending on its predecessor;
// the grid lines of a mesh in natural order).
//
// One CTA per right-hand side / system, one thread per line. Step s solves
// every row whose level is s: a thread solves at most one row per step, the
// dependency on its own previous row stays in a register and dependencies on
// other lines are read from a shared-memory ring holding each line's last
// `window` values, so one step costs a barrier plus a short chain of shared
// loads and fp64 operations. Everything a step consumes is staged ahead with
// cp.async: the schedule (dependency descriptors + factor values, laid out
// [step][entry][thread]) as one contiguous block per batch of K steps copied
// by the whole CTA, and each thread's vector operands (its line's rows are
// consecutive) up to 2K rows ahead. The wait happens once per batch, not per
// level (tools/microbench_level.cu: a per-level wait costs 150-200 cycles).
//
// Summation order and unfused fp64 arithmetic are those of the reference
// (sparse.py:222-239), so results are bit-identical to pcgkit.
#include <algorithm>

#include "trsv.cuh"

namespace npcg {

namespace {

__device__ __forceinline__ unsigned smem_addr(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cpa8(void *dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cpa_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void line_epilogue(const LineArgs &a, int b, double total) {
    if (a.upper) bwd_epilogue(a.st, b, total);
    else fwd_epilogue(a.st, b, total, a.drift_count);
}

}  // namespace

template <int MD, bool UPPER, bool PCG, bool SB>
__global__ void __launch_bounds__(1024) trsv_line_kernel(LineArgs a) {
    extern __shared__ __align__(16) char sm[];
    __shared__ double s_red[32];
    const LineDir &L = a.dir;
    const int T = L.T, t = threadIdx.x, K = a.K, VR = 2 * a.K;
    const int b = blockIdx.x;
    // what this system needs from this launch
    int op = TOP_SOLVE;
    if (PCG) {
        const SolveState &st = a.st;
        const int ph = st.status[b] == ST_ACTIVE ? st.phase[b] : -1;
        op = !UPPER ? (ph == PH_ITER ? TOP_UPDATE : (ph == PH_INIT ? TOP_SOLVE : TOP_SKIP))
                    : ((ph == PH_ITER || ph == PH_INIT) ? TOP_SOLVE : TOP_SKIP);
        if (op == TOP_SKIP) {
            if (UPPER && t == 0) line_epilogue(a, b, 0.0);  // keeps pflag / restart bookkeeping
            return;
        }
    }
    // shared memory: ring | desc stages | factor stages | vector ring
    const int W = L.window;
    double *ring = reinterpret_cast<double *>(sm);
    const size_t ring_bytes = ((size_t)T * W + 2) * 8;
    int16_t *sdesc = reinterpret_cast<int16_t *>(sm + ((ring_bytes + 15) & ~size_t(15)));
    const size_t desc_stage = (size_t)K * MD * T;  // elements per stage
    double *sval = reinterpret_cast<double *>(reinterpret_cast<char *>(sdesc) + ((2 * desc_stage * 2 + 15) & ~size_t(15)));
    double *vring = sval + 2 * desc_stage;  // [VR][3][T]
    for (int q = t; q < T * W + 2; q += T) ring[q] = 0.0;  // the padding slot reads +0.0

    const int row0 = L.line_row0[t];
    const int len = row0 < 0 ? 0 : L.line_len[t];
    const int dir = UPPER ? -1 : 1;
    const long long cb = (long long)b * a.cs, rs = a.rs;
    const double *Sb = a.S + (SB ? (size_t)b * L.steps_pad * MD * T : 0);
    const int nb = L.steps_pad / K;
    const double alpha = (!UPPER && PCG && op == TOP_UPDATE) ? a.st.alpha[b] : 0.0;

    auto issue_struct = [&](int j) {  // whole CTA: one contiguous block per batch
        const int16_t *gd = L.desc + (size_t)j * desc_stage;
        int16_t *dd = sdesc + (size_t)(j & 1) * desc_stage;
        for (int q = t; q < (int)(desc_stage / 8); q += T) cpa16(dd + 8 * q, gd + 8 * q);
        const double *gs = Sb + (size_t)j * desc_stage;
        double *ds = sval + (size_t)(j & 1) * desc_stage;
        for (int q = t; q < (int)(desc_stage / 2); q += T) cpa16(ds + 2 * q, gs + 2 * q);
    };
    int k_iss = 0;
    auto issue_vectors = [&](int upto) {  // this thread: rows [k_iss, upto) of its line
        upto = min(upto, len);
        for (; k_iss < upto; ++k_iss) {
            const long long vi = (long long)(row0 + dir * k_iss) * rs + cb;
            double *v = vring + (size_t)(k_iss % VR) * 3 * T + t;
            if (!UPPER) {
                cpa8(v, a.in + vi);  // r
                if (PCG && op == TOP_UPDATE) cpa8(v + T, a.AP + vi);
            } else {
                cpa8(v, a.in + vi);  // y
                cpa8(v + T, a.d_batched ? a.D + vi : a.D + (row0 + dir * k_iss));  // D shared: [n]
                if (PCG) cpa8(v + 2 * T, a.R + vi);
            }
        }
    };

    issue_struct(0);
    issue_vectors(VR);
    cpa_commit();
    double prev = 0.0, acc2 = 0.0;
    int k = 0;  // rows of this line solved so far
    for (int j = 0; j < nb; ++j) {
        cpa_wait_all();
        __syncthreads();  // batch j's schedule and the vectors issued a batch ago have landed
        if (j + 1 < nb) issue_struct(j + 1);
        issue_vectors(k + VR);
        cpa_commit();
        const int16_t *dd = sdesc + (size_t)(j & 1) * desc_stage;
        const double *ds = sval + (size_t)(j & 1) * desc_stage;
        for (int q = 0; q < K; ++q) {
            const int16_t *dq = dd + (size_t)q * MD * T + t;
            const double *sq = ds + (size_t)q * MD * T + t;
            const int d0 = dq[0];
            if (d0 != kNoRow) {
                const double *v = vring + (size_t)(k % VR) * 3 * T + t;
                double acc;
                if (!UPPER) {
                    if (PCG && op == TOP_UPDATE) {  // r -= alpha Ap (pcg.py:142)
                        acc = __dsub_rn(v[0], __dmul_rn(alpha, v[T]));
                        a.R[(long long)(row0 + k) * rs + cb] = acc;
                        acc2 = __dadd_rn(acc2, __dmul_rn(acc, acc));
                    } else {
                        acc = v[0];
                    }
                } else {
                    acc = __ddiv_rn(v[0], v[T]);  // z /= diag (sparse.py:273)
                }
                double y[MD], s[MD];
#pragma unroll
                for (int e = 0; e < MD; ++e) {
                    const int d = e == 0 ? d0 : dq[(size_t)e * T];
                    s[e] = sq[(size_t)e * T];
                    y[e] = d == -1 ? prev : ring[d];
                }
#pragma unroll
                for (int e = 0; e < MD; ++e) acc = __dsub_rn(acc, __dmul_rn(s[e], y[e]));
                if (UPPER && PCG) acc2 = __dadd_rn(acc2, __dmul_rn(v[2 * T], acc));
                prev = acc;
                ring[t * W + (k & (W - 1))] = acc;
                a.out[(long long)(row0 + dir * k) * rs + cb] = acc;
                ++k;
            }
            __syncthreads();  // step done: its values are visible to the next step
        }
    }
    cpa_wait_all();
    if (PCG) {  // fixed-order block reduction of r.r (forward) or r.z (backward)
        double v = acc2;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, off));
        if ((t & 31) == 0) s_red[t >> 5] = v;
        __syncthreads();
        if (t == 0) {
            double tot = 0.0;
            for (int w = 0; w < (T + 31) / 32; ++w) tot = __dadd_rn(tot, s_red[w]);
            line_epilogue(a, b, tot);
        }
    }
}

size_t line_smem_bytes(const LineDir &L, int K) {
    const size_t ring = (((size_t)L.T * L.window + 2) * 8 + 15) & ~size_t(15);
    const size_t st = (size_t)K * L.md * L.T;
    return ring + ((2 * st * 2 + 15) & ~size_t(15)) + 2 * st * 8 + (size_t)2 * K * 3 * L.T * 8;
}

int line_batch_for(const LineDir &L) {
    for (int K : {6, 3, 2, 1})
        if (line_smem_bytes(L, K) <= 200 * 1024) return K;
    return 0;
}

template <int MD, bool UPPER, bool PCG, bool SB>
static cudaError_t launch_line_t(const LineArgs &a, cudaStream_t s) {
    auto kern = trsv_line_kernel<MD, UPPER, PCG, SB>;
    const size_t smem = line_smem_bytes(a.dir, a.K);
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    note_launch();
    kern<<<a.B, a.dir.T, smem, s>>>(a);
    return cudaGetLastError();
}

template <int MD>
static cudaError_t launch_line_md(const LineArgs &a, cudaStream_t s) {
    const bool pcg = a.mode == TRSV_PCG;
    if (a.upper) {
        if (pcg) return a.s_batched ? launch_line_t<MD, true, true, true>(a, s) : launch_line_t<MD, true, true, false>(a, s);
        return a.s_batched ? launch_line_t<MD, true, false, true>(a, s) : launch_line_t<MD, true, false, false>(a, s);
    }
    if (pcg) return a.s_batched ? launch_line_t<MD, false, true, true>(a, s) : launch_line_t<MD, false, true, false>(a, s);
    return a.s_batched ? launch_line_t<MD, false, false, true>(a, s) : launch_line_t<MD, false, false, false>(a, s);
}

cudaError_t launch_trsv_line(const LineArgs &a, cudaStream_t s) {
    switch (a.dir.md) {
        case 2: return launch_line_md<2>(a, s);
        case 3: return launch_line_md<3>(a, s);
        case 4: return launch_line_md<4>(a, s);
        case 8: return launch_line_md<8>(a, s);
        default: return cudaErrorInvalidValue;
    }
}

// packed[b][step][e][t] = S[b][vperm]   (batched: S laid out system-major)
__global__ void line_factor_pack_kernel(long long per, int B, int sb, long long ps, long long bs, const int *vperm,
                                        const double *S, double *packed) {
    const long long total = per * (sb ? B : 1);
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
         q += (long long)gridDim.x * blockDim.x) {
        const long long b = q / per, e = q % per;
        const int p = vperm[e];
        packed[q] = p < 0 ? 0.0 : S[(long long)p * ps + b * bs];
    }
}

void launch_line_factor_pack(const LineDir &L, int B, int sb, long long ps, long long bs, const double *S,
                             double *packed, cudaStream_t s) {
    const long long per = (long long)L.steps_pad * L.md * L.T;
    const long long total = per * (sb ? B : 1);
    note_launch();
    line_factor_pack_kernel<<<(int)std::min<long long>((total + 255) / 256, 16384), 256, 0, s>>>(
        per, B, sb, ps, bs, L.vperm, S, packed);
}

}  // namespace npcg
