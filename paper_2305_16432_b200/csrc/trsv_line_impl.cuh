// trsv_line_impl.cuh -- the line-wavefront P^{-1} kernel and its launch
// templates (see trsv_line.cu). Included by one translation unit per
// (PCG, systems per cluster) pair so the instances compile in parallel.
#pragma once
#include <algorithm>
#include <type_traits>
#include <cstdlib>

#include "ptx.cuh"
#include "trsv.cuh"

namespace npcg {

namespace {


__device__ __forceinline__ double ld_vol(const double *p) { return *reinterpret_cast<const volatile double *>(p); }
__device__ __forceinline__ void st_vol(double *p, double v) { *reinterpret_cast<volatile double *>(p) = v; }
__device__ __forceinline__ bool is_sentinel(double v) {
    return (unsigned long long)__double_as_longlong(v) == kSentinel;
}
__device__ __forceinline__ double sentinel() { return __longlong_as_double((long long)kSentinel); }
// distributed shared memory: address of `p` in CTA `rank` of the cluster
__device__ __forceinline__ unsigned map_rank(const void *p, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ double ld_dsm(unsigned addr) {
    unsigned long long v;
    asm volatile("ld.relaxed.cluster.shared::cluster.b64 %0, [%1];" : "=l"(v) : "r"(addr) : "memory");
    return __longlong_as_double((long long)v);
}
// the same through a generic address (mapa.u64, formed once per warp: the
// per-store window conversion of the shared::cluster form is off the step path)
__device__ __forceinline__ double *map_rank_generic(const void *p, unsigned rank) {
    double *r;
    asm volatile("mapa.u64 %0, %1, %2;" : "=l"(r) : "l"(p), "r"(rank));
    return r;
}
__device__ __forceinline__ double ld_gen(const double *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.cluster.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return __longlong_as_double((long long)v);
}
__device__ __forceinline__ void st_gen(double *p, double v) {
    asm volatile("st.relaxed.cluster.b64 [%0], %1;" ::"l"(p), "l"(__double_as_longlong(v)) : "memory");
}
__device__ __forceinline__ void st_dsm(unsigned addr, double v) {
    asm volatile("st.relaxed.cluster.shared::cluster.b64 [%0], %1;" ::"r"(addr), "l"(__double_as_longlong(v))
                 : "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// element of (step q of a tile, lane t) in a direction's traversal order:
// a lane's steps 2h and 2h+1 are adjacent (pattern.h)
__device__ __forceinline__ int tile_elem(int q, int t) { return (q >> 1) * 64 + t * 2 + (q & 1); }

// sum of u[i] v[i] over a stage's steps in a fixed pairwise order (padding
// steps hold zeros), so the running dot product waits on one add per stage
template <int N>
__device__ __forceinline__ double stage_dot(const double (&u)[N], const double (&v)[N]) {
    double p[N];
#pragma unroll
    for (int i = 0; i < N; ++i) p[i] = __dmul_rn(u[i], v[i]);
#pragma unroll
    for (int h = 1; h < N; h <<= 1)
#pragma unroll
        for (int i = 0; i + h < N; i += 2 * h) p[i] = __dadd_rn(p[i], p[i + h]);
    return p[0];
}

#ifdef NPCG_LINE_TRACE
// Debug timeline (build with -DNPCG_LINE_TRACE): CTA 0 of system 0, per
// warp (line warps, then helpers) and stage, three clock64 stamps, into
// LineArgs::trace ([kTraceWarps][kTraceStages][3]).
#define WS_TRACE(role, jj, k)                                                                    \
    do {                                                                                          \
        if (trace_on && t == 0 && (jj) < kLineTraceStages)                                        \
            io.trace[(((role) * 8 + wl_) * kLineTraceStages + (jj)) * 3 + (k)] = clock64();       \
    } while (0)
#else
#define WS_TRACE(role, jj, k) \
    do {                      \
    } while (0)
#endif

// exact y / D from D and rD = RN(1 / D): q = RN(y rD) is within an ulp of
// the quotient, the residual e = y - q D is exact (FMA), and RN(q + e rD)
// is the correctly rounded quotient (Markstein) -- bitwise __ddiv_rn(y, D),
// three fp64 operations instead of a division sequence. e == 0 means q is
// exact (and keeps the sign of a zero y); quotients near the ends of the
// exponent range, infinities and NaNs take the division.
__device__ __forceinline__ double div_by_diag(double y, double D, double rD) {
    const double q = __dmul_rn(y, rD);
    const double e = __fma_rn(-q, D, y);
    double r = e == 0.0 ? q : __fma_rn(e, rD, q);
    const double aq = fabs(q);
    if (q != 0.0 && !(aq > 0x1p-960 && aq < 0x1p960)) r = __ddiv_rn(y, D);
    return r;
}

// whether div_by_diag's fast path may not be taken for quotient q: integer
// tests on the exponent field (no fp64 compares, no branches); zero is fine,
// exponents outside [2^-959, 2^960), infinities and NaNs are not
__device__ __forceinline__ bool quotient_needs_division(double q) {
    const unsigned hi = (unsigned)__double2hiint(q), lo = (unsigned)__double2loint(q);
    const unsigned ex = (hi >> 20) & 0x7ffu;
    const bool zero = ((hi & 0x7fffffffu) | lo) == 0u;
    return !zero & (ex - 64u > 1918u);
}
__device__ __forceinline__ bool is_zero_bits(double e) {
    return (((unsigned)__double2hiint(e) & 0x7fffffffu) | (unsigned)__double2loint(e)) == 0u;
}

// y / D for many elements at once: the fast path for all of them first (no
// branch between them), then the division for any lane that needs it
// (div_by_diag's range conditions, tested conservatively), once per batch
// and warp
template <int K>
__device__ __forceinline__ void div_by_diag_batch(double2 (&y)[K], const double2 (&d)[K], const double2 (&rd)[K]) {
    bool slow = false;
    double2 q[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double qx = __dmul_rn(y[k].x, rd[k].x), qy = __dmul_rn(y[k].y, rd[k].y);
        const double ex = __fma_rn(-qx, d[k].x, y[k].x), ey = __fma_rn(-qy, d[k].y, y[k].y);
        slow |= quotient_needs_division(qx) | quotient_needs_division(qy);
        const double fx = __fma_rn(ex, rd[k].x, qx), fy = __fma_rn(ey, rd[k].y, qy);
        qx = is_zero_bits(ex) ? qx : fx;
        qy = is_zero_bits(ey) ? qy : fy;
        q[k] = make_double2(qx, qy);
    }
    if (__any_sync(0xffffffffu, slow)) {
#pragma unroll
        for (int k = 0; k < K; ++k) q[k] = make_double2(div_by_diag(y[k].x, d[k].x, rd[k].x), div_by_diag(y[k].y, d[k].y, rd[k].y));
    }
#pragma unroll
    for (int k = 0; k < K; ++k) y[k] = q[k];
}

// A stage slot of a line-warp pair holds G tiles of: the factor kinds
// [G][3][128], then three vector areas [G][128] each:
//   forward:  V0 = r (the helper turns it into r - alpha Ap in place)
//             V1 = Ap, overwritten by the solver's y
//   backward: V0 = y (the helper turns it into y / D in place)
//             V1 = D, overwritten by the solver's z;  V2 = 1 / D
//
// KR right-hand sides per cluster (shared factor only): the factor kinds are
// staged once, the three vector areas once per right-hand side ([KR][3][G][128]
// after the kinds), and the line warp interleaves KR independent dependency
// chains -- one factor load and one stage hand-off serve KR chains. A shared
// diagonal is staged once (into the first right-hand side's areas).
__host__ __device__ constexpr int slot_arrays(int KR) { return kLineKinds + 3 * KR; }
constexpr int kLineMaxKR = 4;

// One direction of the solve for one line warp.
struct LineDirIO {
    const int4 *meta = nullptr;    // this direction's warp table
    const double *fac = nullptr;   // packed factor values of this direction (this system)
    const double *v[3] = {};       // vectors the helper stages (the first system's base; see above)
    long long vstride[3] = {};     // distance between the cluster's systems in each of them (0: shared)
    int nv = 0;                    // how many of them
    double *out = nullptr;         // y (forward) or z (backward)
    double *rg = nullptr;          // forward PCG update: r_{k+1}
    const double *rdot = nullptr;  // backward PCG: r, for r.z
    long long sys = 0;             // distance between the cluster's systems in out / rg / rdot
    double *ring = nullptr;        // this direction's incoming-value rings, [WL][R] in this CTA
    int w = 0;                     // warp in this direction's order
    bool rev = false;              // the direction's warp w runs on line warp W - 1 - w
    int jbase = 0;                 // stages the pair consumed before (mbarrier parity)
    long long *trace = nullptr;    // debug timeline (NPCG_LINE_TRACE builds)
};

// Solver warp: the dependency chains only. Per step a lane reads its
// prepared operands (r_{k+1} or y / D per right-hand side, and the three
// factor kinds) from the slot, takes the left neighbour's values by shuffle
// (lane 0: from the ring written by the previous warp's lane 31), and leaves
// the results in the slot. The KR chains of a step are independent: their
// shuffle / multiply / subtract latencies overlap.
template <bool UPPER, int G, int NS, int KR>
__device__ __forceinline__ void line_solver(const LineDirIO &io, const int W, const int WL, const int R, const int wl,
                                            const int t, uint64_t *full, uint64_t *done, char *slots,
                                            const size_t slot_bytes, const bool trace_on) {
    const int wl_ = wl;
    (void)trace_on;
    (void)wl_;
    constexpr int STEPS = kTileSteps * G;
    static_assert(2 * STEPS <= 32, "a stage pair's ring slots are checked by one warp");
    const int w = io.w;
    const int4 *meta = io.meta;
    const int4 me = meta[w];
    const int C0 = me.x, nt = me.y, C1 = C0 + kTileSteps * nt;
    const int nstage = (nt + G - 1) / G;
    // ring protocol: warp w sends its last lane's values of steps
    // [max(C0_right - 2, C0), min(C1_right - 1, C1)) to the right warp; every
    // value is read once and re-armed by its reader. A ring slot of step x
    // holds the KR chains' values at (x mod R) * KR.
    int P0 = 0, P1 = 0, Q0 = 0, Q1 = 0;
    if (w > 0) {
        const int4 pm = meta[w - 1];
        P0 = pm.x;
        P1 = pm.x + kTileSteps * pm.y;
    }
    if (w + 1 < W) {
        const int4 qm = meta[w + 1];
        Q0 = max(qm.x - 2, C0);
        Q1 = min(qm.x + kTileSteps * qm.y - 1, C1);
    }
    const bool cons = w > 0 && t == 0, prod = w + 1 < W && t == 31;
    double *rin = io.ring + (size_t)wl * R * KR;  // my incoming ring (local)
    // my outgoing ring: the right warp's incoming ring, in its CTA
    const int wr = w + 1 < W ? w + 1 : w;
    const int pr = io.rev ? W - 1 - wr : wr;  // its line warp
    double *rout = map_rank_generic(io.ring + (size_t)(pr % WL) * R * KR, (unsigned)(pr / WL));
    auto out_slot = [&](int x) { return rout + (x & (R - 1)) * KR; };
    double h0[KR], lp[KR], ychk[KR];
#pragma unroll
    for (int c = 0; c < KR; ++c) h0[c] = 0.0, lp[c] = 0.0, ychk[c] = sentinel();
    // h0: my value one step back; lp: left neighbour's value two steps back (at the
    // next step); ychk: this stage pair's outgoing-slot check (loaded a pair ahead)
    if (w + 1 < W) {
        const int ys = C0 + t;
        if (t < 2 * STEPS && ys >= Q0 && ys < Q1 && ys - R >= Q0) {
#pragma unroll
            for (int c = 0; c < KR; ++c) ychk[c] = ld_gen(out_slot(ys) + c);
        }
    }
    if (cons && C0 - 2 >= P0 && C0 - 2 < P1) {  // value of the left line at step C0 - 2 (0 outside its range)
        double *p = rin + ((C0 - 2) & (R - 1)) * KR;
#pragma unroll
        for (int c = 0; c < KR; ++c) {
            double v = ld_vol(p + c);
            while (is_sentinel(v)) {  // start-up: the left warp is a whole line-block ahead
                __nanosleep(64);
                v = ld_vol(p + c);
            }
            st_vol(p + c, sentinel());
            lp[c] = v;
        }
    }
    constexpr size_t kFac = (size_t)G * kLineKinds * kTileSlots, kVec = (size_t)G * kTileSlots;  // doubles
    for (int j = 0; j < nstage; ++j) {
        const int jj = io.jbase + j;
        const int s = jj % NS, sig = C0 + j * STEPS;  // first step of the stage
        const int g = min(G, nt - j * G);
        WS_TRACE(0, jj, 0);
        const int live_steps = g * kTileSteps;
        const double *f = reinterpret_cast<const double *>(slots + (size_t)s * slot_bytes);
        double *vin = const_cast<double *>(f) + kFac;  // chain c: operands at vin + 3 c kVec, results one area on
        // left line's values at steps sig-1 .. sig+STEPS-2 (lane i holds step sig-1+i): one
        // batch per stage, each slot re-armed after the read
        double x[KR];
#pragma unroll
        for (int c = 0; c < KR; ++c) x[c] = 0.0;
        if (w > 0) {
            const int xs = sig - 1 + t;
            const bool pend = t < STEPS && xs >= P0 && xs < P1 && xs < C1 - 1;
            double *px = rin + (xs & (R - 1)) * KR;
            bool miss = false;
            if (pend) {
#pragma unroll
                for (int c = 0; c < KR; ++c) x[c] = ld_vol(px + c), miss |= is_sentinel(x[c]);
            }
            while (__any_sync(0xffffffffu, miss)) {
                __nanosleep(20);
                if (miss) {
                    miss = false;
#pragma unroll
                    for (int c = 0; c < KR; ++c) x[c] = ld_vol(px + c), miss |= is_sentinel(x[c]);
                }
            }
            if (pend) {
#pragma unroll
                for (int c = 0; c < KR; ++c) st_vol(px + c, sentinel());
            }
        }
        WS_TRACE(2, jj, 0);
        // my outgoing slots of this stage pair must have been re-armed by the right warp;
        // checked once per two stages (lane i: step sig + i), loaded two stages ahead (a
        // re-armed slot stays so until I write it)
        if (w + 1 < W && (j & 1) == 0) {
            const int ys = sig + t;
            const bool chk = t < 2 * STEPS && ys >= Q0 && ys < Q1 && ys - R >= Q0;
            const double *py = out_slot(ys);
            auto busy = [&]() {
                bool bz = false;
#pragma unroll
                for (int c = 0; c < KR; ++c) bz |= !is_sentinel(ychk[c]);
                return chk && bz;
            };
            while (__any_sync(0xffffffffu, busy())) {
                __nanosleep(20);
                if (chk) {
#pragma unroll
                    for (int c = 0; c < KR; ++c) ychk[c] = ld_gen(py + c);
                }
            }
            const int yn = ys + 2 * STEPS;  // the next pair's slots
            const bool chn = t < 2 * STEPS && yn >= Q0 && yn < Q1 && yn - R >= Q0;
#pragma unroll
            for (int c = 0; c < KR; ++c) ychk[c] = chn ? ld_gen(out_slot(yn) + c) : sentinel();
        }
        WS_TRACE(2, jj, 1);
        mbar_wait(&full[s], (jj / NS) & 1);  // operands prepared by the helper
        WS_TRACE(0, jj, 1);
        // a step pair's operands (a lane's two steps of a tile half are adjacent, pattern.h:
        // one 16-byte load each), loaded one pair ahead so the shared-memory reads overlap
        // the chain. A partial stage's lookahead reads stale slot contents, never used.
        auto pair_at = [&](int i) {  // element offset of step pair (i, i + 1) in this direction
            const int tp = UPPER ? G - 1 - i / kTileSteps - (G - g) : i / kTileSteps;  // tile within the stage
            const int tpc = tp < 0 ? 0 : tp;
            const int e = tile_elem(i % kTileSteps, t);
            return make_int2(tpc * kLineKinds * kTileSlots + e, tpc * kTileSlots + (UPPER ? kTileSlots - 2 - e : e));
        };
        auto pair_ops = [&](int i, double2 &f0, double2 &f1, double2 &f2, double2 (&a0)[KR]) {
            const int2 o = pair_at(i);
            f0 = *reinterpret_cast<const double2 *>(f + o.x);
            f1 = *reinterpret_cast<const double2 *>(f + o.x + kTileSlots);
            f2 = *reinterpret_cast<const double2 *>(f + o.x + 2 * kTileSlots);
#pragma unroll
            for (int c = 0; c < KR; ++c) a0[c] = *reinterpret_cast<const double2 *>(vin + 3 * c * kVec + o.y);
        };
        // The steps of a stage, specialised on what the stage needs besides the chain:
        // FULL: all G tiles live (no per-pair bound check); SEND 0: nothing goes to the right
        // warp, 1: every step does and the ring slots of the stage do not wrap (one base
        // address, immediate offsets), 2: checked per step.
        auto run = [&](auto full_c, auto send_c) {
            constexpr bool FULL = decltype(full_c)::value;
            constexpr int SEND = decltype(send_c)::value;
            double *obase = out_slot(sig);
            double2 cf0, cf1, cf2, ca0[KR];
            pair_ops(0, cf0, cf1, cf2, ca0);
#pragma unroll
            for (int pi = 0; pi < STEPS / 2; ++pi) {
                const int i = 2 * pi;
                if (!FULL && i >= live_steps) break;
                double2 nf0, nf1, nf2, na0[KR];
                if (pi + 1 < STEPS / 2) pair_ops(i + 2, nf0, nf1, nf2, na0);
                const double F0[2] = {cf0.x, cf0.y}, F1[2] = {cf1.x, cf1.y}, F2[2] = {cf2.x, cf2.y};
                double A[KR][2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {  // sparse.py:222-239 order: L2, L1, S1 terms
                    const int step = sig + i + h;
                    const bool send = SEND == 2 && prod && step >= Q0 && step < Q1;
#pragma unroll
                    for (int c = 0; c < KR; ++c) {
                        // vectors are in forward tile order: the backward pair is reversed
                        const double V = (h == 0) == UPPER ? ca0[c].y : ca0[c].x;
                        const double pre = __dsub_rn(V, __dmul_rn(F0[h], lp[c]));
                        const double p2 = __dmul_rn(F2[h], h0[c]);
                        double l1 = __shfl_up_sync(0xffffffffu, h0[c], 1);
                        const double xl = __shfl_sync(0xffffffffu, x[c], i + h);
                        if (t == 0) l1 = xl;
                        double acc = __dsub_rn(pre, __dmul_rn(F1[h], l1));
                        acc = __dsub_rn(acc, p2);
                        h0[c] = acc;
                        lp[c] = l1;
                        if (SEND == 1) {
                            if (t == 31) st_gen(obase + (i + h) * KR + c, acc);
                        } else if (send) {
                            st_gen(out_slot(step) + c, acc);
                        }
                        A[c][h] = acc;
                    }
                }
                const int2 o = pair_at(i);
#pragma unroll
                for (int c = 0; c < KR; ++c)
                    *reinterpret_cast<double2 *>(vin + (3 * c + 1) * kVec + o.y) =
                        UPPER ? make_double2(A[c][1], A[c][0]) : make_double2(A[c][0], A[c][1]);
                if (pi + 1 < STEPS / 2) {
                    cf0 = nf0, cf1 = nf1, cf2 = nf2;
#pragma unroll
                    for (int c = 0; c < KR; ++c) ca0[c] = na0[c];
                }
            }
        };
        {
            const int last = sig + live_steps - 1;
            const bool right = w + 1 < W;
            const bool none = !right || last < Q0 || sig >= Q1;
            const bool all = right && sig >= Q0 && last < Q1 && (sig & (R - 1)) + live_steps <= R;
            if (g == G && all) run(std::true_type{}, std::integral_constant<int, 1>{});
            else if (g == G && none) run(std::true_type{}, std::integral_constant<int, 0>{});
            else run(std::false_type{}, std::integral_constant<int, 2>{});
        }
        __syncwarp();  // every lane's results are in the slot
        if (t == 0) mbar_arrive(&done[s]);
        WS_TRACE(0, jj, 2);
    }
}

// What a cluster's right-hand sides need from this launch.
template <int KR>
struct LineRhs {
    bool act[KR];      // solved in this launch (results written back)
    bool upd[KR];      // forward phase applies r -= alpha Ap first (PCG iteration)
    double alpha[KR];
};

// Helper warp of a line warp: stages the operands with TMA, prepares them
// (r_{k+1} = r - alpha Ap with |r_{k+1}|^2, pcg.py:142-143; or y / D,
// sparse.py:273), writes the solver's results back to global memory
// (coalesced) and forms r.z (pcg.py:167; r is brought into the slot's 1/D
// area by a second bulk copy once y / D is formed). Adds this lane's dot
// partials to acc[]. Every loop over a stage is unrolled over its 2G chunks
// per lane: the loads of a stage are in flight together. A right-hand side
// that does not iterate in this launch is staged and solved like the others
// (the chains are independent) but nothing of it is written back.
template <bool UPPER, bool PCG, int G, int NS, int KR>
__device__ __forceinline__ void line_helper(const LineDirIO &io, const int t, const LineRhs<KR> &rhs, double (&acc)[KR],
                                            uint64_t *tma, uint64_t *full, uint64_t *done, uint64_t *rtma,
                                            char *slots, const size_t slot_bytes, const int wl_, const bool trace_on) {
    (void)trace_on;
    (void)wl_;
    constexpr int K = 2 * G;  // double2 chunks per lane per stage (g * 64 chunks of a stage)
    const int4 me = io.meta[io.w];
    const int nt = me.y, tile0 = me.z;
    const int nstage = (nt + G - 1) / G;
    auto stage_tiles = [&](int j, int &lo, int &g) {  // ascending in memory; backward walks them downwards
        g = min(G, nt - j * G);
        lo = UPPER ? tile0 + nt - j * G - g : tile0 + j * G;
    };
    constexpr size_t kFac = (size_t)G * kLineKinds * kTileSlots, kVec = (size_t)G * kTileSlots;  // doubles
    auto slot_of = [&](int s) { return reinterpret_cast<double *>(slots + (size_t)s * slot_bytes); };
    // vector v of chain c is staged unless it is shared (stride 0) and c > 0, or (forward)
    // it is Ap of a right-hand side without an update
    auto staged = [&](int c, int v) {
        if (v >= io.nv) return false;
        if (c > 0 && io.vstride[v] == 0) return false;
        if (!UPPER && v == 1 && !rhs.upd[c]) return false;
        return true;
    };
    auto issue = [&](int j) {  // lane 0: bulk copies of stage j into its slot
        int lo, g;
        stage_tiles(j, lo, g);
        const int s = (io.jbase + j) % NS;
        double *sp = slot_of(s);
        const unsigned fb = (unsigned)g * kLineKinds * kTileSlots * 8, vb = (unsigned)g * kTileSlots * 8;
        unsigned nvec = 0;
#pragma unroll
        for (int c = 0; c < KR; ++c)
            for (int v = 0; v < 3; ++v) nvec += staged(c, v) ? 1u : 0u;
        mbar_expect_tx(&tma[s], fb + nvec * vb);
        bulk_g2s(sp, io.fac + (size_t)lo * kLineKinds * kTileSlots, fb, &tma[s]);
#pragma unroll
        for (int c = 0; c < KR; ++c)
            for (int v = 0; v < 3; ++v)
                if (staged(c, v))
                    bulk_g2s(sp + kFac + (3 * c + v) * kVec, io.v[v] + c * io.vstride[v] + (size_t)lo * kTileSlots, vb,
                             &tma[s]);
    };
    if (t == 0)
        for (int j = 0; j < NS && j < nstage; ++j) issue(j);
    int jp = 0, jw = 0;  // next stage to prepare / to write back
    // whatever is ready first, write-backs (they issue the refills) before
    // preparations; never block on one while the other could proceed
    while (jw < nstage) {
        const int jjw = io.jbase + jw, sw = jjw % NS;
        const bool wb_ready = jw < jp && mbar_test(&done[sw], (jjw / NS) & 1) &&
                              (!(UPPER && PCG) || mbar_test(&rtma[sw], (jw / NS) & 1));
        const int jjp = io.jbase + jp;
        const bool prep_ready = !wb_ready && jp < nstage && jp < jw + NS && mbar_test(&tma[jjp % NS], (jjp / NS) & 1);
        if (!wb_ready && !prep_ready) continue;
        if (prep_ready) {
            const int jj = jjp, s = jj % NS;
            WS_TRACE(1, jj, 0);
            int lo, g;
            stage_tiles(jp, lo, g);
            double *sp = slot_of(s);
            const int nc = g * (kTileSlots / 2);
#pragma unroll
            for (int c = 0; c < KR; ++c) {
                double2 *v0 = reinterpret_cast<double2 *>(sp + kFac + 3 * c * kVec);
                if (UPPER) {
                    // a shared diagonal sits in the first chain's areas
                    const int cd = io.vstride[1] == 0 ? 0 : c;
                    const double2 *v1 = reinterpret_cast<const double2 *>(sp + kFac + (3 * cd + 1) * kVec);
                    const double2 *v2 = reinterpret_cast<const double2 *>(sp + kFac + (3 * cd + 2) * kVec);
                    double2 y[K], d[K], rd[K];
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        const int q = t + 32 * k < nc ? t + 32 * k : t;
                        y[k] = v0[q], d[k] = v1[q], rd[k] = v2[q];
                    }
                    div_by_diag_batch<K>(y, d, rd);
#pragma unroll
                    for (int k = 0; k < K; ++k)
                        if (t + 32 * k < nc) v0[t + 32 * k] = y[k];
                } else if (PCG && rhs.upd[c]) {
                    const double2 *v1 = reinterpret_cast<const double2 *>(sp + kFac + (3 * c + 1) * kVec);
                    const double alpha = rhs.alpha[c];
                    double2 r[K], ap[K];
                    double part[K];
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        const int q = t + 32 * k < nc ? t + 32 * k : t;
                        r[k] = v0[q], ap[k] = v1[q];
                    }
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        r[k].x = __dsub_rn(r[k].x, __dmul_rn(alpha, ap[k].x));  // pcg.py:142
                        r[k].y = __dsub_rn(r[k].y, __dmul_rn(alpha, ap[k].y));
                        part[k] = t + 32 * k < nc ? __dadd_rn(__dmul_rn(r[k].x, r[k].x), __dmul_rn(r[k].y, r[k].y)) : 0.0;
                        if (t + 32 * k < nc) {
                            v0[t + 32 * k] = r[k];
                            // r_{k+1} goes to global memory from the registers here (the write-back
                            // would read it from the slot again)
                            if (rhs.act[c]) reinterpret_cast<double2 *>(io.rg + c * io.sys + (size_t)lo * kTileSlots)[t + 32 * k] = r[k];
                        }
                    }
#pragma unroll
                    for (int h = 1; h < K; h <<= 1)  // |r_{k+1}|^2 (pcg.py:143), fixed pairwise order
#pragma unroll
                        for (int k = 0; k + h < K; k += 2 * h) part[k] = __dadd_rn(part[k], part[k + h]);
                    acc[c] = __dadd_rn(acc[c], part[0]);
                }
            }
            __syncwarp();
            if (t == 0) mbar_arrive(&full[s]);
            WS_TRACE(3, jj, 0);
            if (UPPER && PCG) {  // r for r.z into the 1/D areas, no longer read
                fence_proxy_async();
                __syncwarp();
                if (t == 0) {
                    const unsigned vb = (unsigned)g * kTileSlots * 8;
                    mbar_expect_tx(&rtma[s], KR * vb);
#pragma unroll
                    for (int c = 0; c < KR; ++c)
                        bulk_g2s(sp + kFac + (3 * c + 2) * kVec, io.rdot + c * io.sys + (size_t)lo * kTileSlots, vb,
                                 &rtma[s]);
                }
            }
            WS_TRACE(1, jj, 1);
            ++jp;
        } else {
            const int jj = jjw, s = sw;  // rtma is armed in this phase only: parity by jw
            (void)jj;
            int lo, g;
            stage_tiles(jw, lo, g);
            const double *sp = slot_of(s);
            const int nc = g * (kTileSlots / 2);
            // everything the write-back needs leaves the slot first, so the refill (the head of
            // the slot's done -> refill -> prepare chain) is issued before the global stores
            double2 res[KR][K], rk[KR][K];
#pragma unroll
            for (int c = 0; c < KR; ++c) {
                const double2 *v0 = reinterpret_cast<const double2 *>(sp + kFac + 3 * c * kVec);
                const double2 *v1 = reinterpret_cast<const double2 *>(sp + kFac + (3 * c + 1) * kVec);
                const double2 *v2 = reinterpret_cast<const double2 *>(sp + kFac + (3 * c + 2) * kVec);
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const int q = t + 32 * k < nc ? t + 32 * k : t;
                    res[c][k] = v1[q];
                    if (UPPER && PCG) rk[c][k] = v2[q];
                }
            }
            // the slot's generic accesses (mine and the solver's) before the async-proxy refill
            fence_proxy_async();
            __syncwarp();
            if (t == 0 && jw + NS < nstage) issue(jw + NS);
#pragma unroll
            for (int c = 0; c < KR; ++c) {
                if (!rhs.act[c]) continue;
                double2 *og = reinterpret_cast<double2 *>(io.out + c * io.sys + (size_t)lo * kTileSlots);
                double part[K];
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const bool ok = t + 32 * k < nc;
                    if (ok) og[t + 32 * k] = res[c][k];  // y | z
                    part[k] = (UPPER && PCG && ok) ? __dadd_rn(__dmul_rn(rk[c][k].x, res[c][k].x), __dmul_rn(rk[c][k].y, res[c][k].y)) : 0.0;
                }
                if (UPPER && PCG) {  // r.z (pcg.py:167), fixed pairwise order
#pragma unroll
                    for (int h = 1; h < K; h <<= 1)
#pragma unroll
                        for (int k = 0; k + h < K; k += 2 * h) part[k] = __dadd_rn(part[k], part[k + h]);
                    acc[c] = __dadd_rn(acc[c], part[0]);
                }
            }
            WS_TRACE(1, jj, 2);
            ++jw;
        }
    }
}



}  // namespace

// P^{-1} r for KR systems per cluster, one launch: the forward unit solve
// (with the PCG residual update in front), then y / D and the backward
// transpose solve (sparse.py:222-239, 265-275; pcg.py:142-143, 167).
//
// Warps come in pairs (line warp w: warp w of the CTA, its helper: warp
// WL + w): the line warp carries only the wavefront's dependency chains, the
// helper everything else (line_helper). Every line warp owns the same 32
// grid lines in both directions (the backward order walks warp W-1-w, lane
// 31-t), so the backward operands of a pair's rows are values its own
// helper wrote in the forward phase: a proxy fence and the helper's TMA
// loads carry them over, no grid-wide barrier. The backward wavefront starts
// on the last warp as soon as it finishes its forward rows.
//
// PCG mode is speculative across the phase boundary: the backward solve runs
// for every system that iterates; the forward epilogue (which may turn the
// system to the drift check, pcg.py:147) runs before the backward one at the
// end, and the backward epilogue then ignores the solve (common.cuh).
//
// WB bounds the line warps per CTA (launch bounds: 4 pairs = 256 threads keep
// the full register file per thread, 8 pairs get 128 registers).
template <bool PCG, bool SB, int G, int NS, int C, int KR, int WB>
__global__ void __launch_bounds__(64 * WB, 1) ldlt_line_kernel(LineArgs a) {
    static_assert(KR == 1 || !SB, "several right-hand sides per cluster share one factor");
    extern __shared__ __align__(128) char sm[];
    __shared__ double s_red[2][KR][kLineMaxWarps];
    __shared__ double s_cta[2][KR][4];
    // WL line warps (+ WL helpers) per CTA; the last CTA of a cluster may hold idle pairs
    const int W = a.warps, WL = (W + C - 1) / C, R = a.ring;
    const int warp = threadIdx.x >> 5, t = threadIdx.x & 31;
    const bool helper = warp >= WL;
    const int wl = helper ? warp - WL : warp;
    const int rank = C > 1 ? (int)cluster_rank() : 0, b0 = (blockIdx.x / C) * KR;
    const int pw = rank * WL + wl;  // line warp = forward warp
    const bool idle = pw >= W;
    // what the cluster's systems need from this launch (uniform over the cluster)
    LineRhs<KR> rhs;
    bool any = !PCG;
#pragma unroll
    for (int c = 0; c < KR; ++c) {
        rhs.act[c] = !PCG;
        rhs.upd[c] = false;
        rhs.alpha[c] = 0.0;
        if (PCG) {
            const SolveState &st = a.st;
            const int ph = st.status[b0 + c] == ST_ACTIVE ? st.phase[b0 + c] : -1;
            rhs.upd[c] = ph == PH_ITER;
            rhs.act[c] = ph == PH_ITER || ph == PH_INIT;
            any |= rhs.act[c];
        }
    }
    if (PCG && !any) {
        // every thread of the cluster has read status / phase before the
        // epilogue changes them (PH_RESTART -> PH_INIT)
        if (C > 1) cluster_sync_all();
        else __syncthreads();
        if (rank == 0 && threadIdx.x == 0) {
#pragma unroll
            for (int c = 0; c < KR; ++c) bwd_epilogue(a.st, b0 + c, 0.0);  // pflag / restart bookkeeping
        }
        return;
    }
    if (PCG && helper) {
#pragma unroll
        for (int c = 0; c < KR; ++c)
            if (rhs.upd[c]) rhs.alpha[c] = a.st.alpha[b0 + c];
    }
    const LineSmem m = line_layout(WL, R, G, NS, KR);
    double *ring_f = reinterpret_cast<double *>(sm + m.ring_f);
    double *ring_b = reinterpret_cast<double *>(sm + m.ring_b);
    uint64_t *bars = reinterpret_cast<uint64_t *>(sm + m.bars) + (size_t)wl * 4 * NS;
    uint64_t *tma = bars, *full = bars + NS, *done = bars + 2 * NS, *rtma = bars + 3 * NS;
    char *slots = sm + m.slots + (size_t)wl * NS * m.slot_bytes;
    for (int i = threadIdx.x; i < WL * R * KR; i += blockDim.x) ring_f[i] = ring_b[i] = sentinel();
    if (helper && t == 0) {
        for (int s = 0; s < 4 * NS; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    if (C > 1) cluster_sync_all();  // every ring armed before any remote write
    else __syncthreads();

    const long long vb = (long long)b0 * a.nslot;
    const long long db = a.d_batched ? vb : 0;
    const bool trace_on = b0 == 0 && rank == 0 && a.trace != nullptr;
    const size_t fb = SB ? (size_t)b0 * a.fac_slots : 0;
    double acc_f[KR], acc_b[KR];
#pragma unroll
    for (int c = 0; c < KR; ++c) acc_f[c] = acc_b[c] = 0.0;
    if (!idle) {
        LineDirIO F;
        F.meta = reinterpret_cast<const int4 *>(a.meta_f);
        F.fac = a.S_f + fb;
        F.v[0] = a.in + vb;
        F.v[1] = PCG ? a.AP + vb : nullptr;
        F.vstride[0] = F.vstride[1] = a.nslot;
        F.nv = PCG ? 2 : 1;
        F.out = a.Y + vb;
        F.rg = PCG ? a.R + vb : nullptr;
        F.sys = a.nslot;
        F.ring = ring_f;
        F.w = pw;
        F.rev = false;
        F.jbase = 0;
        F.trace = a.trace;
        LineDirIO Bk;
        Bk.meta = reinterpret_cast<const int4 *>(a.meta_b);
        Bk.fac = a.S_b + fb;
        Bk.v[0] = a.Y + vb;
        Bk.v[1] = a.D + db;
        Bk.v[2] = a.rD + db;
        Bk.vstride[0] = a.nslot;
        Bk.vstride[1] = Bk.vstride[2] = a.d_batched ? a.nslot : 0;
        Bk.nv = 3;
        Bk.out = a.out + vb;
        Bk.rdot = PCG ? a.R + vb : nullptr;
        Bk.sys = a.nslot;
        Bk.ring = ring_b;
        Bk.w = W - 1 - pw;
        Bk.rev = true;
        Bk.jbase = (F.meta[pw].y + G - 1) / G;
        Bk.trace = a.trace;
        if (helper) {
            line_helper<false, PCG, G, NS, KR>(F, t, rhs, acc_f, tma, full, done, rtma, slots, m.slot_bytes, wl, trace_on);
            // the backward phase reads this warp's y (and r) stores through TMA
            fence_proxy_async_global();
            __syncwarp();
            line_helper<true, PCG, G, NS, KR>(Bk, t, rhs, acc_b, tma, full, done, rtma, slots, m.slot_bytes, wl, trace_on);
        } else {
            line_solver<false, G, NS, KR>(F, W, WL, R, wl, t, full, done, slots, m.slot_bytes, trace_on);
            line_solver<true, G, NS, KR>(Bk, W, WL, R, wl, t, full, done, slots, m.slot_bytes, trace_on);
        }
    }
    if (PCG) {  // fixed-order reductions: lanes, helper warps, then the cluster's CTAs
#pragma unroll
        for (int c = 0; c < KR; ++c) {
            double vf = acc_f[c], vbk = acc_b[c];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                vf = __dadd_rn(vf, __shfl_down_sync(0xffffffffu, vf, off));
                vbk = __dadd_rn(vbk, __shfl_down_sync(0xffffffffu, vbk, off));
            }
            if (helper && t == 0) s_red[0][c][wl] = vf, s_red[1][c][wl] = vbk;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
#pragma unroll
            for (int c = 0; c < KR; ++c) {
                double tf = 0.0, tb = 0.0;
                for (int q = 0; q < WL; ++q) tf = __dadd_rn(tf, s_red[0][c][q]), tb = __dadd_rn(tb, s_red[1][c][q]);
                if (C > 1) {
                    st_dsm(map_rank(&s_cta[0][c][rank], 0), tf);
                    st_dsm(map_rank(&s_cta[1][c][rank], 0), tb);
                } else {
                    fwd_epilogue(a.st, b0 + c, tf, a.drift_count);
                    bwd_epilogue(a.st, b0 + c, tb);
                }
            }
        }
    }
    if (C > 1) {  // remote rings / partials stay valid until every CTA of the cluster is done
        cluster_sync_all();
        if (PCG && rank == 0 && threadIdx.x == 0) {
#pragma unroll
            for (int c = 0; c < KR; ++c) {
                double tf = 0.0, tb = 0.0;
                for (int q = 0; q < C; ++q) tf = __dadd_rn(tf, s_cta[0][c][q]), tb = __dadd_rn(tb, s_cta[1][c][q]);
                fwd_epilogue(a.st, b0 + c, tf, a.drift_count);
                bwd_epilogue(a.st, b0 + c, tb);
            }
        }
    }
}

template <bool PCG, bool SB, int G, int NS, int C, int KR, int WB>
static cudaError_t launch_ldlt_w(const LineArgs &a, cudaStream_t s) {
    auto kern = ldlt_line_kernel<PCG, SB, G, NS, C, KR, WB>;
    const int WL = (a.warps + C - 1) / C;
    const size_t smem = line_layout(WL, a.ring, G, NS, KR).total;
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    note_launch();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.B / KR * C);
    cfg.blockDim = dim3(64 * WL);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a);
}

template <bool PCG, bool SB, int G, int NS, int C, int KR>
static cudaError_t launch_ldlt_t(const LineArgs &a, cudaStream_t s) {
    if constexpr (C == 2) {
        return launch_ldlt_w<PCG, SB, G, NS, C, KR, line_cta_warps(2)>(a, s);
    } else {
        const int WL = (a.warps + C - 1) / C;
        if (WL <= 4) return launch_ldlt_w<PCG, SB, G, NS, C, KR, 4>(a, s);
        if constexpr (C == 4 && KR == 1) {  // 513-line grids (config 3): 5 pairs, 204 registers
            if (WL <= 5) return launch_ldlt_w<PCG, SB, G, NS, C, KR, 5>(a, s);
        }
        return launch_ldlt_w<PCG, SB, G, NS, C, KR, kLineMaxWarps>(a, s);
    }
}

template <bool PCG, int KR, int G, int NS, int C>
static cudaError_t launch_ldlt_gc(const LineArgs &a, cudaStream_t s) {
    if constexpr (KR == 1) {
        if (a.s_batched) return launch_ldlt_t<PCG, true, G, NS, C, 1>(a, s);
    }
    if (a.s_batched) return cudaErrorInvalidValue;  // several systems per cluster share the factor
    return launch_ldlt_t<PCG, false, G, NS, C, KR>(a, s);
}

template <bool PCG, int KR, int C>
static cudaError_t launch_ldlt_c(const LineArgs &a, cudaStream_t s) {
    switch (a.group * 16 + a.stages) {
        case 4 * 16 + 2: return launch_ldlt_gc<PCG, KR, 4, 2, C>(a, s);
        case 3 * 16 + 3: return launch_ldlt_gc<PCG, KR, 3, 3, C>(a, s);
        case 2 * 16 + 4: return launch_ldlt_gc<PCG, KR, 2, 4, C>(a, s);
        case 2 * 16 + 3: return launch_ldlt_gc<PCG, KR, 2, 3, C>(a, s);
        case 1 * 16 + 4: return launch_ldlt_gc<PCG, KR, 1, 4, C>(a, s);
        default: return cudaErrorInvalidValue;
    }
}

// every kernel of one (PCG, KR) pair: one translation unit each (trsv_line_k*.cu)
template <bool PCG, int KR>
static cudaError_t launch_ldlt_inst(const LineArgs &a, cudaStream_t s) {
    switch (a.cluster) {
        case 1: return launch_ldlt_c<PCG, KR, 1>(a, s);
        case 2: return launch_ldlt_c<PCG, KR, 2>(a, s);
        default: return launch_ldlt_c<PCG, KR, 4>(a, s);
    }
}

}  // namespace npcg
