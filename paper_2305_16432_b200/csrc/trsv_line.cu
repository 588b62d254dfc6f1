// trsv_line.cu -- line-wavefront triangular solves (pattern.h, LineSched).
//
// One system per cluster of C CTAs (C = 1, 2 or 4, each on its own SM), one
// lane per grid line, no block-wide synchronisation inside the solve; the
// forward solve, the diagonal scaling and the backward solve run in ONE
// launch (ldlt_line_kernel):
//
//   * at every step a lane solves the next row of its line. Its operands are
//     its own previous value (register), and its left neighbour's values one
//     and two steps back: one __shfl_up_sync per step (the two-steps-back
//     value is last step's shuffle). Lane 0 of a warp gets them from a
//     shared-memory ring in its own CTA, written by lane 31 of the previous
//     warp -- through distributed shared memory when that warp sits on the
//     other SM of the cluster. A slot holds a NaN sentinel until written and
//     is re-armed by its reader, so an aligned 8-byte value is its own flag:
//     no fence, no counter. Both sides move whole stages: the reader checks
//     and re-arms a stage's slots at once, the writer checks once per stage
//     that its slots were re-armed (a ring spans twice the natural start
//     offset of adjacent warps, so this never waits in the steady state).
//   * each warp streams its own operands: per stage of G tiles (4 steps x 32
//     lanes each) one elected lane issues bulk copies (TMA, cp.async.bulk +
//     one mbarrier per stage) of the factor values and vector slices into the
//     warp's private stage ring. Results go from registers to global memory
//     in coalesced 256-byte warp stores.
//   * the diagonal scaling y /= diag (sparse.py:273) is formed by the
//     backward phase as it reads its operands (off the dependency chain),
//     exactly, from staged D and 1/D (div_by_diag). PCG mode also fuses the
//     forward r -= alpha Ap (pcg.py:142) with |r|^2 (pcg.py:143) and the
//     backward r.z (pcg.py:167), reduced in a fixed order at the end.
//   * splitting a system over C SMs divides what every SM's shared-memory /
//     L1 data path carries per step (operands in, results out), which is
//     what bounds the step rate.
//
// Summation order and unfused fp64 arithmetic are those of the reference
// (sparse.py:222-239): a row's dependencies in the reference's order are a
// subsequence of (L2, L1, S1) and absent kinds carry a zero factor, whose
// product with a finite operand leaves the row sum unchanged, so results are
// bit-identical to pcgkit (up to the sign of an exactly-zero row sum).
#include <algorithm>
#include <cstdlib>

#include "ptx.cuh"
#include "trsv.cuh"

namespace npcg {

static long long *g_trace = nullptr;  // device timeline buffer (NPCG_LINE_TRACE builds)

long long *line_trace_buffer() {
#ifdef NPCG_LINE_TRACE
    if (!g_trace) {
        const size_t bytes = (size_t)kLineTraceWarps * kLineTraceStages * 3 * sizeof(long long);
        if (cudaMalloc(&g_trace, bytes) != cudaSuccess) return nullptr;
        cudaMemset(g_trace, 0, bytes);
    }
#endif
    return g_trace;
}

int line_trace_copy(long long *out, int n) {
#ifdef NPCG_LINE_TRACE
    n = std::min(n, kLineTraceWarps * kLineTraceStages * 3);
    if (!g_trace) return (int)cudaErrorInvalidValue;
    return (int)cudaMemcpy(out, g_trace, n * sizeof(long long), cudaMemcpyDeviceToHost);
#else
    (void)out;
    (void)n;
    return 0;  // no timeline in this build
#endif
}

static size_t line_smem(int WL, int R, int G, int NS, int KR) { return line_smem_bytes(WL, R, G, NS, KR); }

int line_config_for(const LineSched &L, int B, int KR) {
    if (KR < 1 || KR > kLineMaxKR || (KR != 1 && KR != 2 && KR != 4) || B % KR != 0) return 0;
    int dev = 0, optin = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (optin <= 0) optin = 227 * 1024;
    const size_t cap = (size_t)optin - 1024;  // static shared memory
    const int W = L.fwd.warps, R = std::max(L.fwd.ring, L.bwd.ring);
    const int NC = B / KR;  // clusters
    auto fits = [&](int c) { return (W + c - 1) / c <= line_cta_warps(c) && (c == 1 || W >= c); };
    // shapes in order of preference: 12-step stages three deep first (the
    // helper's write-back -> refill -> prepare chain of a slot has two stages
    // of slack instead of one: 116 vs 124 us per launch at config 2 against
    // 16-step stages two deep; 8-step stages four deep: 128 us), then what
    // fits
    static const int prefs[][2] = {{3, 3}, {4, 2}, {2, 4}, {2, 3}, {1, 4}};
    auto shape_for = [&](int c) {
        const int WL = (W + c - 1) / c;
        if (const char *env = std::getenv("NPCG_LINE_CFG")) {
            const int v = std::atoi(env), G = v / 16, NS = v % 16;
            if (line_shape_ok(G, NS) && line_smem(WL, R, G, NS, KR) <= cap) return v;
        }
        for (const auto &p : prefs)
            if (line_smem(WL, R, p[0], p[1], KR) <= cap) return p[0] * 16 + p[1];
        return 0;
    };
    // CTAs per system: split over two SMs while the batch leaves them free;
    // more than 8 line warps always take a cluster (2 CTAs up to 16 warps,
    // 4 beyond; the last CTA may hold idle pairs)
    int C = (W % 2 == 0 && 2 * NC <= sms && fits(2)) ? 2 : 1;
    if (!fits(C)) C = (fits(2) && 2 * NC <= sms) ? 2 : 4;
    // several right-hand sides per cluster need more shared memory per pair:
    // spread the pairs over more CTAs while that buys longer stages
    if (KR > 1 && C < 4 && fits(4) && 4 * NC <= sms && shape_for(4) / 16 > shape_for(C) / 16) C = 4;
    if (const char *env = std::getenv("NPCG_LINE_CLUSTER")) {
        const int c = std::atoi(env);
        if ((c == 1 || c == 2 || c == 4) && fits(c)) C = c;
    }
    if (!fits(C)) C = fits(2) ? 2 : (fits(4) ? 4 : 0);
    if (!C) return 0;
    int shape = shape_for(C);
    if (!shape && C < 4 && fits(4)) shape = shape_for(C = 4);
    if (!shape) return 0;
    return (KR << 16) | (C * 256 + shape);
}

cudaError_t launch_ldlt_line(const LineArgs &a, cudaStream_t s) {
    if (!line_shape_ok(a.group, a.stages) || a.warps < 1 || (a.cluster != 1 && a.cluster != 2 && a.cluster != 4) ||
        (a.warps + a.cluster - 1) / a.cluster > line_cta_warps(a.cluster) ||
        (a.kr != 1 && a.kr != 2 && a.kr != 4) || a.B % a.kr != 0)
        return cudaErrorInvalidValue;
    LineArgs b = a;
    b.trace = line_trace_buffer();
    const bool pcg = a.mode == TRSV_PCG;
    switch (a.kr) {
        case 1: return pcg ? launch_ldlt_k1p(b, s) : launch_ldlt_k1n(b, s);
        case 2: return pcg ? launch_ldlt_k2p(b, s) : launch_ldlt_k2n(b, s);
        default: return pcg ? launch_ldlt_k4p(b, s) : launch_ldlt_k4n(b, s);
    }
}

__global__ void reciprocal_kernel(long long count, const double *D, double *rD) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < count; q += (long long)gridDim.x * blockDim.x)
        rD[q] = __ddiv_rn(1.0, D[q]);
}

cudaError_t launch_reciprocal(long long count, const double *D, double *rD, cudaStream_t s) {
    if (count <= 0) return cudaSuccess;
    note_launch();
    reciprocal_kernel<<<(int)std::min<long long>((count + 255) / 256, 4096), 256, 0, s>>>(count, D, rD);
    return cudaGetLastError();
}

// packed[b][e] = S[vperm[e] * ps + b * bs]
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
    const long long per = L.fac_slots;
    const long long total = per * (sb ? B : 1);
    note_launch();
    line_factor_pack_kernel<<<(int)std::min<long long>((total + 255) / 256, 16384), 256, 0, s>>>(
        per, B, sb, ps, bs, L.vperm, S, packed);
}

}  // namespace npcg
