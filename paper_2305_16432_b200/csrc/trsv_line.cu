// trsv_line.cu -- line-wavefront triangular solves for patterns whose rows
// form at most kLineMaxLines "lines" (runs of rows each depending on its
// predecessor; the grid lines of a mesh in natural order).
//
// One CTA per right-hand side / system, warp-specialised:
//
//   consumers (threads 0..T-1, one per line) walk the steps. At step s every
//     line whose rigid step range covers s solves one row: the dependency
//     on its own previous row is a register, the cross-line ones are read
//     from a shared-memory ring holding every line's last `window` values.
//     A step is a handful of shared loads, an unfused fp64 chain and one
//     named barrier over the consumer warps -- nothing else.
//   producers (kProdWarps warps) move whole batches of kLineBatch steps.
//     Every vector lives in line order (pattern.h), so a batch's rows are one
//     contiguous slot range: one elected producer bulk-copies (TMA,
//     cp.async.bulk + mbarrier) the batch's schedule block, factor values
//     and vector slices into a stage ring, the producer warps form the
//     right-hand sides slot by slot (r - alpha Ap forward, y / diag
//     backward) and, once the consumers are done, accumulate the PCG dot
//     product and bulk-store the solved slices back (TMA store). No thread
//     issues a scattered global access.
//
// Stage hand-off uses named barriers: FULL[s] (producers arrive, consumers
// sync) and EMPTY[s] (consumers arrive, producers sync), so a consumer pays
// one barrier per step plus one per batch.
//
// Summation order and unfused fp64 arithmetic are those of the reference
// (sparse.py:222-239), so results are bit-identical to pcgkit.
#include <algorithm>

#ifndef NPCG_NO_ZERO_Y
#define NPCG_NO_ZERO_Y 0
#endif
#include "ptx.cuh"
#include "trsv.cuh"

namespace npcg {

namespace {

constexpr int kProdWarps = 8;
constexpr int kProd = 32 * kProdWarps;
constexpr int kLineMaxStages = 6;
constexpr int kBarCons = 1;
constexpr int kBarFull = 2;
constexpr int kBarEmpty = kBarFull + kLineMaxStages;
constexpr int kBarProd = kBarEmpty + kLineMaxStages;
constexpr int kPrefetchBatches = 0;  // L2 prefetch distance of the bulk copies

struct LineSmem {  // byte offsets into dynamic shared memory
    size_t ring, stage0, stage_bytes, sv, v[3], meta, total;
};

__host__ __device__ inline size_t al128(size_t x) { return (x + 127) & ~size_t(127); }

__host__ __device__ inline LineSmem line_layout(int T, int W, int MD, int maxs, int NS, int nv, int nb) {
    LineSmem m;
    m.ring = 128;  // mbarriers first
    m.stage0 = al128(m.ring + ((size_t)T * W + 2) * 8);
    size_t o = al128(16 + (size_t)maxs * MD * 2);  // schedule block
    m.sv = o;
    o = al128(o + (size_t)maxs * MD * 8);
    for (int i = 0; i < 3; ++i) {
        m.v[i] = o;
        if (i < nv) o = al128(o + (size_t)maxs * 8);
    }
    m.stage_bytes = o;
    m.meta = m.stage0 + NS * o;  // per batch: boff | bslot | bcount
    m.total = m.meta + (size_t)nb * 16;
    return m;
}

__device__ __forceinline__ void line_epilogue(const LineArgs &a, int b, double total) {
    if (a.upper) bwd_epilogue(a.st, b, total);
    else fwd_epilogue(a.st, b, total, a.drift_count);
}

}  // namespace

// Debug timeline of CTA 0 of the forward solve (build with -DNPCG_LINE_TRACE):
// clock64 per batch and event, read back with npcg_debug_line_trace().
constexpr int kTraceEvents = 16, kTraceBatches = 2048;
__device__ long long g_line_trace[kTraceEvents][kTraceBatches];
#ifdef NPCG_LINE_TRACE
#define LTRACE(ev, j)                                                                                     \
    do {                                                                                                  \
        if (!UPPER && blockIdx.x == 0 && (j) < kTraceBatches) g_line_trace[ev][j] = clock64();            \
    } while (0)
#else
#define LTRACE(ev, j) \
    do {              \
    } while (0)
#endif

template <int MD, bool UPPER, bool PCG, bool SB>
__global__ void __launch_bounds__(kLineMaxLines + kProd, 1) trsv_line_kernel(LineArgs a) {
    constexpr int K = kLineBatch;
    extern __shared__ __align__(128) char sm[];
    __shared__ double s_red[kProdWarps];
    const LineDir &L = a.dir;
    const int T = L.T, NS = a.stages, W = L.window, nb = L.nbatch;
    const int tid = threadIdx.x, b = blockIdx.x;
    const int NT = T + kProd;  // threads taking part in FULL / EMPTY
    // what this system needs from this launch
    int op = TOP_SOLVE;
    if (PCG) {
        const SolveState &st = a.st;
        const int ph = st.status[b] == ST_ACTIVE ? st.phase[b] : -1;
        op = !UPPER ? (ph == PH_ITER ? TOP_UPDATE : (ph == PH_INIT ? TOP_SOLVE : TOP_SKIP))
                    : ((ph == PH_ITER || ph == PH_INIT) ? TOP_SOLVE : TOP_SKIP);
        if (op == TOP_SKIP) {
            if (UPPER && tid == 0) line_epilogue(a, b, 0.0);  // keeps pflag / restart bookkeeping
            return;
        }
    }
    const bool upd = !UPPER && PCG && op == TOP_UPDATE;
    const int nv = UPPER ? (PCG ? 3 : 2) : 2;
    const LineSmem m = line_layout(T, W, MD, L.max_slots, NS, nv, nb);
    uint64_t *mbar = reinterpret_cast<uint64_t *>(sm);
    double *ring = reinterpret_cast<double *>(sm + m.ring);  // [W][T] + zero cell
    auto stage_ptr = [&](int s) { return sm + m.stage0 + (size_t)s * m.stage_bytes; };
    for (int q = tid; q < T * W + 2; q += blockDim.x) ring[q] = 0.0;
    long long *s_boff = reinterpret_cast<long long *>(sm + m.meta);
    int *s_bslot = reinterpret_cast<int *>(s_boff + nb), *s_bcount = s_bslot + nb;
    for (int q = tid; q < nb; q += blockDim.x) {
        s_boff[q] = L.boff[q];
        s_bslot[q] = L.bslot[q];
        s_bcount[q] = L.bcount[q];
    }
    if (tid == T) {
        for (int s = 0; s < NS; ++s) mbar_init(&mbar[s], 1);
        fence_mbar_init();
    }
    __syncthreads();

    if (tid < T) {
        // ------------------------------------------------------------------ consumers
        const int t = tid, len = L.line_len[t], lst = L.line_start[t];
        double prev = 0.0;
        for (int j = 0; j < nb; ++j) {
            const int s = j % NS;
            const int s_cnt_j = s_bcount[j];
            if (t == 0) LTRACE(0, j);
            bar_sync(kBarFull + s, NT);  // stage s holds batch j (also orders the last step's ring writes)
            if (t == 0) LTRACE(1, j);
            char *sp = stage_ptr(s);
            const int *hdr = reinterpret_cast<const int *>(sp);
            const int cnt = s_cnt_j;
            const int16_t *dsc = reinterpret_cast<const int16_t *>(sp) + 8;
            const double *sv = reinterpret_cast<const double *>(sp + m.sv);
            double *vin = reinterpret_cast<double *>(sp + m.v[0]);                // rhs (r / y/D)
            double *vout = reinterpret_cast<double *>(sp + m.v[UPPER ? 0 : 1]);   // solution
#pragma unroll
            for (int q = 0; q < K; ++q) {
                const int kp = j * K + q - lst;  // position of this line's row solved at this step
                if ((unsigned)kp < (unsigned)len) {
                    const int u = hdr[q] + t;
                    int d[MD];
                    double v[MD];
#pragma unroll
                    for (int e = 0; e < MD; ++e) {
                        d[e] = dsc[e * cnt + u];
                        v[e] = sv[e * cnt + u];
                    }
                    double acc = vin[u];
                    double y[MD];
#pragma unroll
                    for (int e = 0; e < MD; ++e) y[e] = d[e] == -1 ? prev : ring[d[e]];
#pragma unroll
                    for (int e = 0; e < MD; ++e) acc = __dsub_rn(acc, __dmul_rn(v[e], y[e]));
                    prev = acc;
                    ring[(kp & (W - 1)) * T + t] = acc;
                    vout[u] = acc;
                }
                if (t == 0) LTRACE(8 + q, j);
                if (q + 1 < K) bar_sync(kBarCons, T);  // step done: its values are visible to the next step
            }
            if (t == 0) LTRACE(2, j);
            fence_proxy_async();            // solution writes -> the producers' TMA store (async proxy)
            bar_arrive(kBarEmpty + s, NT);  // batch j's solution is in stage s
        }
        return;
    }

    // ---------------------------------------------------------------------- producers
    const int p = tid - T;  // 0 .. kProd-1
    const bool elect = p == 0;
    const long long vb = (long long)b * a.nslot;
    const double *Sb = a.S + (SB ? (size_t)b * L.fac_slots : 0);
    const double *Db = a.D + (a.d_batched ? vb : 0);
    const double alpha = upd ? a.st.alpha[b] : 0.0;
    double acc2 = 0.0;
    // sources of batch mb's stage blocks (global)
    auto blocks = [&](int mb, const void **src, unsigned *bytes, int &nsrc) {
        const int bs = s_bslot[mb], cnt = s_bcount[mb];
        const long long bo = s_boff[mb];
        nsrc = 0;
        src[nsrc] = L.sched + bo;
        bytes[nsrc++] = 16 + (unsigned)cnt * MD * 2;
        src[nsrc] = Sb + (bo - 8ll * mb);
        bytes[nsrc++] = (unsigned)cnt * MD * 8;
        src[nsrc] = a.in + vb + bs;
        bytes[nsrc++] = cnt * 8;
        if (!UPPER) {
            if (upd) {
                src[nsrc] = a.AP + vb + bs;
                bytes[nsrc++] = cnt * 8;
            }
        } else {
            src[nsrc] = Db + bs;
            bytes[nsrc++] = cnt * 8;
            if (PCG) {
                src[nsrc] = a.R + vb + bs;
                bytes[nsrc++] = cnt * 8;
            }
        }
    };
    auto issue_load = [&](int mb) {  // elected producer: TMA of batch mb into its stage
        const void *src[5];
        unsigned bytes[5];
        int nsrc;
        blocks(mb, src, bytes, nsrc);
        char *sp = stage_ptr(mb % NS);
        char *dst[5] = {sp, sp + m.sv, sp + m.v[0], sp + m.v[1], sp + m.v[2]};
        unsigned tot = 0;
        for (int i = 0; i < nsrc; ++i) tot += bytes[i];
        uint64_t *bar = &mbar[mb % NS];
        mbar_expect_tx(bar, tot);
        for (int i = 0; i < nsrc; ++i) bulk_g2s(dst[i], src[i], bytes[i], bar);
    };
    auto prefetch = [&](int mb) {
        const void *src[5];
        unsigned bytes[5];
        int nsrc;
        blocks(mb, src, bytes, nsrc);
        for (int i = 0; i < nsrc; ++i) bulk_prefetch_l2(src[i], bytes[i]);
    };
    // batch mb is solved: dot product, then the solved slices go home
    auto drain = [&](int mb) {
        bar_sync(kBarEmpty + mb % NS, NT);
        char *sp = stage_ptr(mb % NS);
        const int bs = s_bslot[mb], cnt = s_bcount[mb];
        if (UPPER && PCG) {  // r.z (pcg.py:167)
            const double *z = reinterpret_cast<const double *>(sp + m.v[0]);
            const double *r = reinterpret_cast<const double *>(sp + m.v[2]);
            for (int u = p; u < cnt; u += kProd) acc2 = __dadd_rn(acc2, __dmul_rn(r[u], z[u]));
        }
        if (elect) {
            fence_proxy_async();  // (every writer fenced before the barriers above)
            if (!UPPER) {
                if (upd) bulk_s2g(a.R + vb + bs, sp + m.v[0], cnt * 8);  // r_{k+1}
                bulk_s2g(a.out + vb + bs, sp + m.v[1], cnt * 8);          // y
            } else {
                bulk_s2g(a.out + vb + bs, sp + m.v[0], cnt * 8);  // z
            }
            bulk_commit();
        }
    };
    constexpr int D = 2;            // batch j - D is drained at iteration j
    const int A = NS - D - 1 > 0 ? NS - D - 1 : 0;
    if (elect) {
        for (int mb = 0; mb < kPrefetchBatches && mb < nb; ++mb) prefetch(mb);

        for (int mb = 0; mb < A && mb < nb; ++mb) issue_load(mb);
    }
    for (int j = 0; j < nb; ++j) {
        if (p == 0) LTRACE(3, j);
        if (j >= D) drain(j - D);
        if (p == 0) LTRACE(4, j);
        const int mb = j + A;
        if (elect && mb < nb) {
            // the stage of batch mb last held mb - NS, drained at iteration mb - NS + D
            if (mb - NS + D >= j) bulk_wait_read<0>();
            else bulk_wait_read<1>();
            issue_load(mb);
            if (kPrefetchBatches > 0 && mb + kPrefetchBatches < nb) prefetch(mb + kPrefetchBatches);
        }
        const int s = j % NS;
        mbar_wait(&mbar[s], (j / NS) & 1);  // batch j's blocks have landed
        if (p == 0) LTRACE(6, j);
        char *sp = stage_ptr(s);
        const int cnt = s_bcount[j];
        if (upd) {  // r -= alpha Ap (pcg.py:142), r.r of the new residual
            double *r = reinterpret_cast<double *>(sp + m.v[0]);
            const double *ap = reinterpret_cast<const double *>(sp + m.v[1]);
            for (int u = p; u < cnt; u += kProd) {
                const double rn = __dsub_rn(r[u], __dmul_rn(alpha, ap[u]));
                r[u] = rn;
                acc2 = __dadd_rn(acc2, __dmul_rn(rn, rn));
            }
        } else if (!UPPER && !NPCG_NO_ZERO_Y) {  // y is written into the (unloaded) second slice: padding slots must read 0
            double2 *y = reinterpret_cast<double2 *>(sp + m.v[1]);
            for (int u = p; u < cnt / 2; u += kProd) y[u] = make_double2(0.0, 0.0);
        } else {  // z /= diag (sparse.py:273)
            double *y = reinterpret_cast<double *>(sp + m.v[0]);
            const double *dg = reinterpret_cast<const double *>(sp + m.v[1]);
            for (int u = p; u < cnt; u += kProd) y[u] = __ddiv_rn(y[u], dg[u]);
        }
        if (p == 0) LTRACE(5, j);
        if (!UPPER) fence_proxy_async();  // r_{k+1} / zeroed y writes -> their TMA store
        bar_arrive(kBarFull + s, NT);
    }
    for (int mb = std::max(0, nb - D); mb < nb; ++mb) drain(mb);
    if (elect) bulk_wait<0>();  // solved slices written before the CTA retires
    if (PCG) {  // fixed-order reduction over the producer threads
        double v = acc2;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, off));
        if ((p & 31) == 0) s_red[p >> 5] = v;
        bar_sync(kBarProd, kProd);
        if (p == 0) {
            double tot = 0.0;
            for (int w = 0; w < kProdWarps; ++w) tot = __dadd_rn(tot, s_red[w]);
            line_epilogue(a, b, tot);
        }
    }
}

int line_trace_copy(long long *out, int n) {
    n = std::min(n, kTraceEvents * kTraceBatches);
    return (int)cudaMemcpyFromSymbol(out, g_line_trace, n * sizeof(long long));
}

size_t line_smem_bytes(const LineDir &L, int stages, bool upper, bool pcg) {
    return line_layout(L.T, L.window, L.md, L.max_slots, stages, upper ? (pcg ? 3 : 2) : 2, L.nbatch).total;
}

int line_stages_for(const LineDir &L, bool upper) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (optin <= 0) optin = 227 * 1024;
    const size_t cap = (size_t)optin - 1024;  // static shared memory
    for (int ns = kLineMaxStages; ns >= 2; --ns)
        if (line_smem_bytes(L, ns, upper, true) <= cap) return ns;
    return 0;
}

template <int MD, bool UPPER, bool PCG, bool SB>
static cudaError_t launch_line_t(const LineArgs &a, cudaStream_t s) {
    auto kern = trsv_line_kernel<MD, UPPER, PCG, SB>;
    const size_t smem = line_smem_bytes(a.dir, a.stages, UPPER, PCG);
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    note_launch();
    kern<<<a.B, a.dir.T + kProd, smem, s>>>(a);
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
    if (a.stages < 2 || a.stages > kLineMaxStages) return cudaErrorInvalidValue;
    switch (a.dir.md) {
        case 2: return launch_line_md<2>(a, s);
        case 3: return launch_line_md<3>(a, s);
        case 4: return launch_line_md<4>(a, s);
        case 8: return launch_line_md<8>(a, s);
        default: return cudaErrorInvalidValue;
    }
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
