// trsv.cu -- the two triangular solves of P^{-1} = (I+L')^{-T} D^{-1} (I+L')^{-1}
// (reference: pkg/src/pcgkit/sparse.py:222-239, 265-275), level-pipelined
// for sm_100a.
//
//   forward : y_i = r_i - sum_{j<i} L'_ij y_j          rows ascending
//   backward: z_j = y_j / D_j - sum_{i>j} L'_ij z_i    rows descending
//
// Work unit = (chunk of contiguous rows, group of G batch columns). One CTA
// owns a unit and walks the chunk's levels with ONE __syncthreads per level.
// Per level it needs (a) the level's schedule block (rows, entry offsets,
// dependency operands, foreign-row list) and factor values -- contiguous,
// 16-byte padded, moved by one TMA bulk copy 2*PD levels ahead into a stage
// ring and signalled on an mbarrier -- and (b) the vectors of the level's
// rows, gathered with cp.async PD levels ahead. Solved values of the last
// `window` levels live in a shared-memory ring. Values owned by earlier
// chunks are published with relaxed stores over a sentinel NaN and staged
// like (b); a still-unsolved staged copy falls back to polling the value
// (no fences, no flags). Every sum keeps the reference's order with
// unfused fp64 operations, so results match sparse.py bit for bit.
#include <algorithm>

#include "ptx.cuh"
#include "trsv.cuh"

namespace npcg {

static __device__ __noinline__ double wait_value(const double *p) {
    long long v = ld_relaxed_b64(p);
    while (v == (long long)kSentinel) v = ld_relaxed_b64(p);
    return __longlong_as_double(v);
}

// ---- per-column control ---------------------------------------------------------
__device__ __forceinline__ int trsv_col_op(const TrsvArgs &a, int b) {
    if (a.mode == TRSV_PLAIN) return TOP_SOLVE;
    const SolveState &st = a.st;
    if (st.status[b] != ST_ACTIVE) return TOP_SKIP;
    const int ph = st.phase[b];
    if (!a.upper) return ph == PH_ITER ? TOP_UPDATE : (ph == PH_INIT ? TOP_SOLVE : TOP_SKIP);
    if (ph == PH_ITER || ph == PH_INIT) return TOP_SOLVE;
    return ph == PH_RESTART ? TOP_RESET : TOP_SKIP;  // forward wrote y: re-arm it
}

__device__ __forceinline__ void trsv_epilogue(const TrsvArgs &a, int b, double total) {
    if (a.upper) bwd_epilogue(a.st, b, total);
    else fwd_epilogue(a.st, b, total, a.drift_count);
}

// ---- the kernel -----------------------------------------------------------------
template <int G, bool UPPER, bool PCG, bool SB>
struct Trsv {
    static constexpr int PD = kTrsvPD;
    static constexpr int NS = 2 * PD + 1;  // level L is read while L+2PD is landing
    static constexpr int ND = PD + 1;
    static constexpr int VS = SB ? G : 1;  // factor values per entry in a stage
    static constexpr int XW = G == 1 ? 2 : G;  // doubles per foreign-value slot

    struct Ctx {
        const TrsvArgs &a;
        const TrsvSmem &m;
        char *sm;
        const int *woff;   // chunk's level table: block word offsets
        const int4 *meta;  // nrow, ne, nx, factor offset
        int g, L0, nl, uop;
    };

    static __device__ __forceinline__ char *struct_stage(const Ctx &c, int ll) {
        return c.sm + c.m.struct_off + (unsigned)(ll % NS) * c.m.struct_bytes;
    }
    static __device__ __forceinline__ double *data_stage(const Ctx &c, int ll) {
        return reinterpret_cast<double *>(c.sm + c.m.data_off + (unsigned)(ll % ND) * c.m.data_bytes);
    }
    static __device__ __forceinline__ uint64_t *mbar(const Ctx &c, int ll) {
        return reinterpret_cast<uint64_t *>(c.sm + c.m.mbar_off) + ll % NS;
    }

    // one thread: TMA the schedule block + factor values of local level ll
    static __device__ __forceinline__ void issue_struct(const Ctx &c, int ll) {
        const int4 mt = c.meta[ll];
        const unsigned wbytes = (unsigned)(c.woff[ll + 1] - c.woff[ll]) * 4u;
        const unsigned sbytes = (unsigned)((mt.y + 1) & ~1) * VS * 8u;
        char *dst = struct_stage(c, ll);
        uint64_t *bar = mbar(c, ll);
        mbar_expect_tx(bar, wbytes + sbytes);
        bulk_g2s(dst, c.a.sched.packed + c.woff[ll], wbytes, bar);
        if (sbytes) {
            const double *src = SB ? c.a.S + ((size_t)c.g * c.a.sched.padded_entries + mt.w) * G : c.a.S + mt.w;
            bulk_g2s(dst + c.m.sval_off, src, sbytes, bar);
        }
    }

    // all threads: gather the vectors of local level ll (its struct has landed)
    static __device__ __forceinline__ void issue_data(const Ctx &c, int ll) {
        const TrsvArgs &a = c.a;
        const int4 mt = c.meta[ll];
        const int nrow = mt.x, nx = mt.z;
        const int *blk = reinterpret_cast<const int *>(struct_stage(c, ll));
        const int *rows = blk;
        const int *xrow = blk + ((nrow + 3) & ~3) + ((nrow + 4) & ~3) + ((mt.y + 3) & ~3);
        double *dv = data_stage(c, ll);
        const int slab = c.m.slab;
        const int B = a.B;
        const size_t cb = (size_t)c.g * G;
        if (c.uop != TOP_SKIP) {
            constexpr int PER = G == 1 ? 1 : 2;  // lanes per copy
            const int units = nrow * (G / PER);
            for (int t = threadIdx.x; t < units; t += kTrsvThreads) {
                const int q = t / (G / PER), l = (t % (G / PER)) * PER;
                const size_t vi = (size_t)rows[q] * B + cb + l;
                double *d0 = dv + q * G + l;
                auto cp = [&](double *dst, const double *src) {
                    if (G == 1) cp_async8(dst, src);
                    else cp_async16(dst, src);
                };
                if (!UPPER) {
                    cp(d0, a.in + vi);  // r (PCG: in == R)
                    if (PCG && c.uop == TOP_UPDATE) cp(d0 + slab, a.AP + vi);
                } else {
                    cp(d0, a.in + vi);
                    if (a.d_batched) cp(d0 + slab, a.D + vi);
                    else if (l == 0) cp_async8(d0 + slab, a.D + rows[q]);
                    if (PCG) cp(d0 + 2 * slab, a.R + vi);
                }
            }
        }
        // foreign values: whatever is published now (16-byte, L2-only copies)
        double *ext = dv + c.m.ext_off;
        const int xunits = nx * (G == 1 ? 1 : G / 2);
        for (int t = threadIdx.x; t < xunits; t += kTrsvThreads) {
            const int x = G == 1 ? t : t / (G / 2), l = G == 1 ? 0 : (t % (G / 2)) * 2;
            const double *src = a.out + (size_t)xrow[x] * B + cb + l;
            if (G == 1) src = reinterpret_cast<const double *>(reinterpret_cast<uintptr_t>(src) & ~uintptr_t(15));
            cp_async16(ext + x * XW + l, src);
        }
    }

    static __device__ void run(const TrsvArgs &a, const TrsvSmem &m, char *sm) {
        __shared__ int s_unit, s_last;
        __shared__ int s_op[kMaxGroup];
        __shared__ double s_red[kTrsvThreads];
        const int tid = threadIdx.x;
        const int B = a.B;
        const int lane = tid % G;  // kTrsvThreads % G == 0
        const Schedule &S = a.sched;
        double *ring = reinterpret_cast<double *>(sm + m.ring_off);
        int *woff = reinterpret_cast<int *>(sm + m.lvl_off);
        int4 *meta = reinterpret_cast<int4 *>(sm + m.lvl_off + (((unsigned)m.lvl_n + 4) & ~3u) * 4u);
        const int ring_span = S.window * S.maxw;

        for (;;) {
            if (tid == 0) s_unit = atomicAdd(&a.ctl->next_unit, 1);
            __syncthreads();
            const int u = s_unit;
            if (u >= a.units) {
                if (tid == 0 && atomicAdd(&a.ctl->exited, 1) == (int)gridDim.x - 1) {
                    a.ctl->next_unit = 0;  // every CTA has fetched its last unit
                    a.ctl->exited = 0;
                }
                return;
            }
            const int cidx = u / a.groups, g = u % a.groups;
            if (tid < G) {
                const int b = g * G + tid;
                s_op[tid] = b < B ? trsv_col_op(a, b) : TOP_SKIP;
            }
            __syncthreads();
            const int b = g * G + lane;
            const int op = s_op[lane];
            int uop = TOP_SKIP;  // what the group's vectors need staged: update > solve > nothing
            for (int q = 0; q < G; ++q) {
                if (s_op[q] == TOP_UPDATE) uop = TOP_UPDATE;
                else if (s_op[q] == TOP_SOLVE && uop != TOP_UPDATE) uop = TOP_SOLVE;
            }
            const bool any = __syncthreads_or(op != TOP_SKIP);
            double acc2 = 0.0;
            if (any) {
                const int L0 = S.chunk_lvl[cidx], nl = S.chunk_lvl[cidx + 1] - L0;
                for (int q = tid; q <= nl; q += kTrsvThreads) woff[q] = S.lvl_woff[L0 + q];
                for (int q = tid; q < nl; q += kTrsvThreads) meta[q] = reinterpret_cast<const int4 *>(S.lvl_meta)[L0 + q];
                if (tid == 0) {
                    for (int s = 0; s < NS; ++s) mbar_init(reinterpret_cast<uint64_t *>(sm + m.mbar_off) + s, 1);
                    fence_proxy_async();
                }
                __syncthreads();
                const Ctx c{a, m, sm, woff, meta, g, L0, nl, uop};
                if (tid == 0)
                    for (int l = 0; l < 2 * PD && l < nl; ++l) issue_struct(c, l);
                for (int l = 0; l < PD; ++l) {  // prologue: vectors of the first PD levels
                    if (l < nl) {
                        mbar_wait(mbar(c, l), 0);
                        issue_data(c, l);
                    }
                    cp_async_commit();
                }
                int ring_base = 0;
                for (int ll = 0; ll < nl; ++ll) {
                    cp_async_wait<PD - 1>();  // this thread's copies of level ll landed
                    __syncthreads();          // ... everyone's; level ll-1 fully solved
                    if (tid == 0 && ll + 2 * PD < nl) {
                        fence_proxy_async();
                        issue_struct(c, ll + 2 * PD);
                    }
                    if (ll + PD < nl) {
                        mbar_wait(mbar(c, ll + PD), (unsigned)((ll + PD) / NS) & 1u);
                        issue_data(c, ll + PD);
                    }
                    cp_async_commit();
                    // ---- solve level ll ----
                    const int4 mt = meta[ll];
                    const int nrow = mt.x;
                    const int *blk = reinterpret_cast<const int *>(struct_stage(c, ll));
                    const int *rows = blk;
                    const int *eoff = blk + ((nrow + 3) & ~3);
                    const int *dep = eoff + ((nrow + 4) & ~3);
                    const int *xrow = dep + ((mt.y + 3) & ~3);
                    const double *sv = reinterpret_cast<const double *>(struct_stage(c, ll) + m.sval_off);
                    const double *dv = data_stage(c, ll);
                    const double *ext = dv + m.ext_off;
                    const int slab = m.slab;
                    if (op != TOP_SKIP) {
                        for (int it = tid; it < nrow * G; it += kTrsvThreads) {
                            const int q = it / G;
                            const int i = rows[q];
                            const size_t vi = (size_t)i * B + b;
                            if (UPPER && PCG && op == TOP_RESET) {  // y of a drifted column: re-arm it
                                reinterpret_cast<long long *>(a.in)[vi] = (long long)kSentinel;
                                continue;
                            }
                            double acc;
                            if (!UPPER) {
                                if (PCG && op == TOP_UPDATE) {  // r -= a Ap (pcg.py:142); x += a p is in pupd
                                    const double al = a.st.alpha[b];
                                    acc = __dsub_rn(dv[it], __dmul_rn(al, dv[slab + it]));
                                    a.R[vi] = acc;
                                    acc2 = __dadd_rn(acc2, __dmul_rn(acc, acc));
                                } else {
                                    acc = dv[it];
                                }
                            } else {
                                const double dd = a.d_batched ? dv[slab + it] : dv[slab + q * G];
                                acc = __ddiv_rn(dv[it], dd);
                                if (PCG)  // consumed: re-arm y for the next forward solve
                                    reinterpret_cast<long long *>(a.in)[vi] = (long long)kSentinel;
                            }
                            const int e1 = eoff[q + 1];
                            for (int e = eoff[q]; e < e1; ++e) {
                                const int d = dep[e];
                                const double s = sv[e * VS + (SB ? lane : 0)];
                                double yj;
                                if (d >= 0) {
                                    yj = ring[d * G + lane];
                                } else {
                                    const int x = -d - 1;
                                    const double *src = a.out + (size_t)xrow[x] * B + b;
                                    yj = ext[x * XW + (G == 1 ? (int)((reinterpret_cast<uintptr_t>(src) >> 3) & 1) : lane)];
                                    if (__double_as_longlong(yj) == (long long)kSentinel) yj = wait_value(src);
                                }
                                acc = __dsub_rn(acc, __dmul_rn(s, yj));
                            }
                            if (UPPER && PCG) acc2 = __dadd_rn(acc2, __dmul_rn(dv[2 * slab + it], acc));
                            ring[(ring_base + q) * G + lane] = acc;
                            st_relaxed_f64(a.out + vi, acc);
                        }
                    }
                    ring_base += S.maxw;
                    if (ring_base >= ring_span) ring_base = 0;
                }
                cp_async_wait<0>();
                __syncthreads();
            }
            // per-unit partial (fixed order: threads with the same lane, ascending)
            if (PCG) {
                s_red[tid] = acc2;
                __syncthreads();
                if (tid < G) {
                    double s = 0.0;
                    for (int t = tid; t < kTrsvThreads; t += G) s = __dadd_rn(s, s_red[t]);
                    a.partial[(size_t)u * G + tid] = s;
                }
            }
            __threadfence();
            __syncthreads();
            if (tid == 0) s_last = atomicAdd(&a.ctl->done, 1) == a.units - 1;
            __syncthreads();
            if (s_last) {
                __threadfence();
                if (PCG) {
                    for (int bb = tid; bb < B; bb += kTrsvThreads) {
                        const int gg = bb / G, lq = bb % G;
                        double s = 0.0;
                        for (int cc = 0; cc < S.chunks; ++cc)
                            s = __dadd_rn(s, __ldcg(&a.partial[((size_t)cc * a.groups + gg) * G + lq]));
                        trsv_epilogue(a, bb, s);
                    }
                }
                if (tid == 0) a.ctl->done = 0;
                __threadfence();
            }
            __syncthreads();
        }
    }
};

template <int G, bool UPPER, bool PCG, bool SB>
__global__ void __launch_bounds__(kTrsvThreads) trsv_kernel(TrsvArgs a, TrsvSmem m) {
    extern __shared__ __align__(128) char sm[];
    Trsv<G, UPPER, PCG, SB>::run(a, m, sm);
}

// ---- host side ------------------------------------------------------------------
static unsigned a16(size_t x) { return (unsigned)((x + 15) & ~size_t(15)); }

TrsvSmem trsv_smem_plan(const Schedule &S, int G, int s_batched) {
    constexpr int PD = kTrsvPD, NS = 2 * PD + 1, ND = PD + 1;
    TrsvSmem m;
    const int vs = s_batched ? G : 1;
    const int xw = G == 1 ? 2 : G;
    m.lvl_n = S.max_chunk_levels + 1;
    size_t off = 0;
    m.ring_off = (unsigned)off;
    off = a16(off + (size_t)S.window * S.maxw * G * 8);
    m.lvl_off = (unsigned)off;
    off = a16(off + (size_t)((m.lvl_n + 4) & ~3) * 4 + (size_t)m.lvl_n * 16);
    m.mbar_off = (unsigned)off;
    off = a16(off + NS * 8);
    m.sval_off = (int)a16((size_t)S.max_words * 4);
    m.struct_bytes = (int)a16(m.sval_off + (size_t)S.max_se * vs * 8);
    off = (off + 127) & ~size_t(127);
    m.struct_off = (unsigned)off;
    off += (size_t)NS * m.struct_bytes;
    m.slab = S.maxw * G;
    m.ext_off = 4 * m.slab;  // in doubles, after 4 vector slabs
    m.data_bytes = (int)a16(((size_t)4 * m.slab + (size_t)S.maxx * xw) * 8);
    m.data_off = (unsigned)off;
    off += (size_t)ND * m.data_bytes;
    m.total = (unsigned)off;
    return m;
}

template <int G, bool UPPER, bool PCG, bool SB>
static cudaError_t launch_t(const TrsvArgs &a, const TrsvSmem &m, cudaStream_t s) {
    auto kern = trsv_kernel<G, UPPER, PCG, SB>;
    static unsigned configured = 0;
    if (m.total > 48 * 1024 && m.total > configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)m.total);
        if (e != cudaSuccess) return e;
        configured = m.total;
    }
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kTrsvThreads, m.total);
    if (per_sm < 1) per_sm = 1;
    const int grid = std::max(1, std::min(a.units, per_sm * num_sms()));
    note_launch();
    kern<<<grid, kTrsvThreads, m.total, s>>>(a, m);
    return cudaGetLastError();
}

template <int G>
static cudaError_t launch_g(const TrsvArgs &a, const TrsvSmem &m, cudaStream_t s) {
    const bool pcg = a.mode == TRSV_PCG;
    if (a.upper) {
        if (pcg) return a.s_batched ? launch_t<G, true, true, true>(a, m, s) : launch_t<G, true, true, false>(a, m, s);
        return a.s_batched ? launch_t<G, true, false, true>(a, m, s) : launch_t<G, true, false, false>(a, m, s);
    }
    if (pcg) return a.s_batched ? launch_t<G, false, true, true>(a, m, s) : launch_t<G, false, true, false>(a, m, s);
    return a.s_batched ? launch_t<G, false, false, true>(a, m, s) : launch_t<G, false, false, false>(a, m, s);
}

cudaError_t launch_trsv(const TrsvArgs &a, cudaStream_t s) {
    const TrsvSmem m = trsv_smem_plan(a.sched, a.G, a.s_batched);
    switch (a.G) {
        case 1: return launch_g<1>(a, m, s);
        case 2: return launch_g<2>(a, m, s);
        case 4: return launch_g<4>(a, m, s);
        case 8: return launch_g<8>(a, m, s);
        default: return cudaErrorInvalidValue;
    }
}

// packed[(g*Ep + e)*G + l] = S[sperm[e]*B + g*G + l]   (batched)
// packed[e]               = S[sperm[e]]                (shared)
__global__ void factor_pack_kernel(long long Ep, int B, int G, int sb, const int *sperm, const double *S,
                                   double *packed) {
    const long long total = sb ? Ep * ((B + G - 1) / G) * G : Ep;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
         q += (long long)gridDim.x * blockDim.x) {
        long long e;
        int b;
        if (sb) {
            const int g = (int)(q / (Ep * G));
            const long long r = q % (Ep * G);
            e = r / G;
            b = g * G + (int)(r % G);
            if (b >= B) {
                packed[q] = 0.0;
                continue;
            }
        } else {
            e = q;
            b = 0;
        }
        const int p = sperm[e];
        packed[q] = p < 0 ? 0.0 : (sb ? S[(size_t)p * B + b] : S[p]);
    }
}

void launch_factor_pack(const Schedule &sched, int B, int G, int sb, const double *S, double *packed,
                        cudaStream_t s) {
    const long long Ep = sched.padded_entries;
    if (Ep <= 0) return;
    const int groups = (B + G - 1) / G;
    const long long total = sb ? Ep * groups * G : Ep;
    note_launch();
    factor_pack_kernel<<<(int)std::min<long long>((total + 255) / 256, 16384), 256, 0, s>>>(Ep, sb ? B : 1, G, sb,
                                                                                           sched.sperm, S, packed);
}

__global__ void fill_sentinel_kernel(long long count, double *p) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < count;
         q += (long long)gridDim.x * blockDim.x)
        reinterpret_cast<long long *>(p)[q] = (long long)kSentinel;
}

void launch_fill_sentinel(long long count, double *p, cudaStream_t s) {
    if (count <= 0) return;
    note_launch();
    fill_sentinel_kernel<<<(int)std::min<long long>((count + 255) / 256, 16384), 256, 0, s>>>(count, p);
}

}  // namespace npcg
