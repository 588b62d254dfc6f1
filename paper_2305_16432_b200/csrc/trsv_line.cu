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

namespace {

// operand stages per warp (a slot is refilled the stage after its use): three
// up to 3-tile stages, two for 4-tile stages (shared memory)
// (tiles per stage, stages in flight) combinations the kernel is built for
__host__ __device__ constexpr bool line_shape_ok(int G, int NS) {
    return (G == 4 && NS == 2) || (G == 2 && (NS == 3 || NS == 4)) || (G == 1 && NS == 4);
}

__host__ __device__ inline size_t al128(size_t x) { return (x + 127) & ~size_t(127); }

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
// warp (line warps, then helpers) and stage, three clock64 stamps.
constexpr int kTraceWarps = 4 * 8, kTraceStages = 1024;
__device__ long long g_ws_trace[kTraceWarps][kTraceStages][3];
#define WS_TRACE(role, jj, k)                                                                             \
    do {                                                                                                   \
        if (trace_on && t == 0 && (jj) < kTraceStages) g_ws_trace[(role) * 8 + wl_][(jj)][(k)] = clock64(); \
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

// y / D for many elements at once: the fast path for all of them first (no
// branch between them), then the division for any lane that needs it
// (div_by_diag's range conditions), once per batch and warp
template <int K>
__device__ __forceinline__ void div_by_diag_batch(double2 (&y)[K], const double2 (&d)[K], const double2 (&rd)[K]) {
    bool slow = false;
    double2 q[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double qx = __dmul_rn(y[k].x, rd[k].x), qy = __dmul_rn(y[k].y, rd[k].y);
        const double ex = __fma_rn(-qx, d[k].x, y[k].x), ey = __fma_rn(-qy, d[k].y, y[k].y);
        const double ax = fabs(qx), ay = fabs(qy);
        slow |= (qx != 0.0 && !(ax > 0x1p-960 && ax < 0x1p960)) || (qy != 0.0 && !(ay > 0x1p-960 && ay < 0x1p960));
        qx = ex == 0.0 ? qx : __fma_rn(ex, rd[k].x, qx);
        qy = ey == 0.0 ? qy : __fma_rn(ey, rd[k].y, qy);
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
constexpr int kSlotArrays = kLineKinds + 3;

// One direction of the solve for one line warp.
struct LineDirIO {
    const int4 *meta = nullptr;    // this direction's warp table
    const double *fac = nullptr;   // packed factor values of this direction (this system)
    const double *v[3] = {};       // vectors the helper stages (this system's base; see above)
    int nv = 0;                    // how many of them
    double *out = nullptr;         // y (forward) or z (backward)
    double *rg = nullptr;          // forward PCG update: r_{k+1}
    const double *rdot = nullptr;  // backward PCG: r, for r.z
    double *ring = nullptr;        // this direction's incoming-value rings, [WL][R] in this CTA
    int w = 0;                     // warp in this direction's order
    bool rev = false;              // the direction's warp w runs on line warp W - 1 - w
    int jbase = 0;                 // stages the pair consumed before (mbarrier parity)
};

// Solver warp: the dependency chain only. Per step a lane reads its
// prepared operands (r_{k+1} or y / D, and the three factor kinds) from the
// slot, takes the left neighbour's value by shuffle (lane 0: from the ring
// written by the previous warp's lane 31), and leaves the result in the slot.
template <bool UPPER, int G, int NS>
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
    // value is read once and re-armed by its reader
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
    double *rin = io.ring + wl * R;  // my incoming ring (local)
    // my outgoing ring: the right warp's incoming ring, in its CTA
    const int wr = w + 1 < W ? w + 1 : w;
    const int pr = io.rev ? W - 1 - wr : wr;  // its line warp
    const unsigned rout = map_rank(io.ring + (pr % WL) * R, (unsigned)(pr / WL));
    auto ring_read = [&](int x) -> double {  // value of the left line at step x (0 outside its range)
        if (x < P0 || x >= P1) return 0.0;
        double *p = rin + (x & (R - 1));
        double v = ld_vol(p);
        while (is_sentinel(v)) {  // start-up: the left warp is a whole line-block ahead
            __nanosleep(64);
            v = ld_vol(p);
        }
        st_vol(p, sentinel());
        return v;
    };
    double h0 = 0.0;  // my value one step back
    double lp = 0.0;  // left neighbour's value two steps back (at the next step)
    double ychk = sentinel();  // this stage pair's outgoing-slot check (loaded a pair ahead)
    if (w + 1 < W) {
        const int ys = C0 + t;
        if (t < 2 * STEPS && ys >= Q0 && ys < Q1 && ys - R >= Q0) ychk = ld_dsm(rout + (unsigned)(ys & (R - 1)) * 8u);
    }
    if (cons) lp = ring_read(C0 - 2);
    for (int j = 0; j < nstage; ++j) {
        const int jj = io.jbase + j;
        const int s = jj % NS, sig = C0 + j * STEPS;  // first step of the stage
        const int g = min(G, nt - j * G);
        WS_TRACE(0, jj, 0);
        const int live_steps = g * kTileSteps;
        const double *f = reinterpret_cast<const double *>(slots + (size_t)s * slot_bytes);
        const double *vin = f + G * kLineKinds * kTileSlots;
        double *res = const_cast<double *>(vin) + G * kTileSlots;
        // left line's values at steps sig-1 .. sig+STEPS-2 (lane i holds step sig-1+i): one
        // batch per stage, each slot re-armed after the read
        double x = 0.0;
        if (w > 0) {
            const int xs = sig - 1 + t;
            const bool pend = t < STEPS && xs >= P0 && xs < P1 && xs < C1 - 1;
            double *px = rin + (xs & (R - 1));
            if (pend) x = ld_vol(px);
            while (__any_sync(0xffffffffu, pend && is_sentinel(x))) {
                __nanosleep(20);
                if (pend) x = ld_vol(px);
            }
            if (pend) st_vol(px, sentinel());
        }
        WS_TRACE(2, jj, 0);
        // my outgoing slots of this stage pair must have been re-armed by the right warp;
        // checked once per two stages (lane i: step sig + i), loaded two stages ahead (a
        // re-armed slot stays so until I write it)
        if (w + 1 < W && (j & 1) == 0) {
            const int ys = sig + t;
            const bool chk = t < 2 * STEPS && ys >= Q0 && ys < Q1 && ys - R >= Q0;
            const unsigned py = rout + (unsigned)(ys & (R - 1)) * 8u;
            while (__any_sync(0xffffffffu, chk && !is_sentinel(ychk))) {
                __nanosleep(20);
                if (chk) ychk = ld_dsm(py);
            }
            const int yn = ys + 2 * STEPS;  // the next pair's slots
            const bool chn = t < 2 * STEPS && yn >= Q0 && yn < Q1 && yn - R >= Q0;
            ychk = chn ? ld_dsm(rout + (unsigned)(yn & (R - 1)) * 8u) : sentinel();
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
        auto pair_ops = [&](int i, double2 &f0, double2 &f1, double2 &f2, double2 &a0) {
            const int2 o = pair_at(i);
            f0 = *reinterpret_cast<const double2 *>(f + o.x);
            f1 = *reinterpret_cast<const double2 *>(f + o.x + kTileSlots);
            f2 = *reinterpret_cast<const double2 *>(f + o.x + 2 * kTileSlots);
            a0 = *reinterpret_cast<const double2 *>(vin + o.y);
        };
        double2 cf0, cf1, cf2, ca0;
        pair_ops(0, cf0, cf1, cf2, ca0);
#pragma unroll
        for (int pi = 0; pi < STEPS / 2; ++pi) {
            const int i = 2 * pi;
            if (i >= live_steps) break;
            double2 nf0, nf1, nf2, na0;
            if (pi + 1 < STEPS / 2) pair_ops(i + 2, nf0, nf1, nf2, na0);
            // vectors are in forward tile order: the backward pair is reversed
            const double V[2] = {UPPER ? ca0.y : ca0.x, UPPER ? ca0.x : ca0.y};
            const double F0[2] = {cf0.x, cf0.y}, F1[2] = {cf1.x, cf1.y}, F2[2] = {cf2.x, cf2.y};
            double A[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {  // sparse.py:222-239 order: L2, L1, S1 terms
                const int step = sig + i + h;
                const double pre = __dsub_rn(V[h], __dmul_rn(F0[h], lp));
                const double p2 = __dmul_rn(F2[h], h0);
                double l1 = __shfl_up_sync(0xffffffffu, h0, 1);
                const double xl = __shfl_sync(0xffffffffu, x, i + h);
                if (t == 0) l1 = xl;
                double acc = __dsub_rn(pre, __dmul_rn(F1[h], l1));
                acc = __dsub_rn(acc, p2);
                h0 = acc;
                lp = l1;
                if (prod && step >= Q0 && step < Q1) st_dsm(rout + (unsigned)(step & (R - 1)) * 8u, acc);
                A[h] = acc;
            }
            const int2 o = pair_at(i);
            *reinterpret_cast<double2 *>(res + o.y) = UPPER ? make_double2(A[1], A[0]) : make_double2(A[0], A[1]);
            if (pi + 1 < STEPS / 2) cf0 = nf0, cf1 = nf1, cf2 = nf2, ca0 = na0;
        }
        __syncwarp();  // every lane's results are in the slot
        if (t == 0) mbar_arrive(&done[s]);
        WS_TRACE(0, jj, 2);
    }
}

// Helper warp of a line warp: stages the operands with TMA, prepares them
// (r_{k+1} = r - alpha Ap with |r_{k+1}|^2, pcg.py:142-143; or y / D,
// sparse.py:273), writes the solver's results back to global memory
// (coalesced) and forms r.z (pcg.py:167; r is brought into the slot's 1/D
// area by a second bulk copy once y / D is formed). Returns this lane's dot
// partial. Every loop over a stage is unrolled over its 2G chunks per lane:
// the loads of a stage are in flight together.
template <bool UPPER, bool PCG, int G, int NS>
__device__ __forceinline__ double line_helper(const LineDirIO &io, const int t, const bool upd, const double alpha,
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
    auto issue = [&](int j) {  // lane 0: bulk copies of stage j into its slot
        int lo, g;
        stage_tiles(j, lo, g);
        const int s = (io.jbase + j) % NS;
        double *sp = slot_of(s);
        const unsigned fb = (unsigned)g * kLineKinds * kTileSlots * 8, vb = (unsigned)g * kTileSlots * 8;
        mbar_expect_tx(&tma[s], fb + io.nv * vb);
        bulk_g2s(sp, io.fac + (size_t)lo * kLineKinds * kTileSlots, fb, &tma[s]);
        for (int v = 0; v < io.nv; ++v) bulk_g2s(sp + kFac + v * kVec, io.v[v] + (size_t)lo * kTileSlots, vb, &tma[s]);
    };
    if (t == 0)
        for (int j = 0; j < NS && j < nstage; ++j) issue(j);
    double acc = 0.0;
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
            double2 *v0 = reinterpret_cast<double2 *>(sp + kFac);
            const double2 *v1 = reinterpret_cast<const double2 *>(sp + kFac + kVec);
            const double2 *v2 = reinterpret_cast<const double2 *>(sp + kFac + 2 * kVec);
            const int nc = g * (kTileSlots / 2);
            if (UPPER) {
                double2 y[K], d[K], rd[K];
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const int c = t + 32 * k < nc ? t + 32 * k : t;
                    y[k] = v0[c], d[k] = v1[c], rd[k] = v2[c];
                }
                div_by_diag_batch<K>(y, d, rd);
#pragma unroll
                for (int k = 0; k < K; ++k)
                    if (t + 32 * k < nc) v0[t + 32 * k] = y[k];
            } else if (PCG && upd) {
                double2 r[K], ap[K];
                double part[K];
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const int c = t + 32 * k < nc ? t + 32 * k : t;
                    r[k] = v0[c], ap[k] = v1[c];
                }
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    r[k].x = __dsub_rn(r[k].x, __dmul_rn(alpha, ap[k].x));  // pcg.py:142
                    r[k].y = __dsub_rn(r[k].y, __dmul_rn(alpha, ap[k].y));
                    part[k] = t + 32 * k < nc ? __dadd_rn(__dmul_rn(r[k].x, r[k].x), __dmul_rn(r[k].y, r[k].y)) : 0.0;
                    if (t + 32 * k < nc) v0[t + 32 * k] = r[k];
                }
#pragma unroll
                for (int h = 1; h < K; h <<= 1)  // |r_{k+1}|^2 (pcg.py:143), fixed pairwise order
#pragma unroll
                    for (int k = 0; k + h < K; k += 2 * h) part[k] = __dadd_rn(part[k], part[k + h]);
                acc = __dadd_rn(acc, part[0]);
            }
            __syncwarp();
            if (t == 0) mbar_arrive(&full[s]);
            WS_TRACE(3, jj, 0);
            if (UPPER && PCG) {  // r for r.z into the 1/D area, no longer read
                fence_proxy_async();
                __syncwarp();
                if (t == 0) {
                    const unsigned vb = (unsigned)g * kTileSlots * 8;
                    mbar_expect_tx(&rtma[s], vb);
                    bulk_g2s(sp + kFac + 2 * kVec, io.rdot + (size_t)lo * kTileSlots, vb, &rtma[s]);
                }
            }
            WS_TRACE(1, jj, 1);
            ++jp;
        } else {
            const int jj = jjw, s = sw;  // rtma is armed in this phase only: parity by jw
            int lo, g;
            stage_tiles(jw, lo, g);
            const double *sp = slot_of(s);
            const double2 *v0 = reinterpret_cast<const double2 *>(sp + kFac);
            const double2 *v1 = reinterpret_cast<const double2 *>(sp + kFac + kVec);
            const double2 *v2 = reinterpret_cast<const double2 *>(sp + kFac + 2 * kVec);
            const int nc = g * (kTileSlots / 2);
            double2 res[K], rk[K];
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int c = t + 32 * k < nc ? t + 32 * k : t;
                res[k] = v1[c];
                if (!UPPER && PCG) rk[k] = v0[c];
                if (UPPER && PCG) rk[k] = v2[c];
            }
            double2 *og = reinterpret_cast<double2 *>(io.out + (size_t)lo * kTileSlots);
            double part[K];
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const bool ok = t + 32 * k < nc;
                if (ok) og[t + 32 * k] = res[k];  // y | z
                if (!UPPER && PCG && upd && ok) reinterpret_cast<double2 *>(io.rg + (size_t)lo * kTileSlots)[t + 32 * k] = rk[k];
                part[k] = (UPPER && PCG && ok) ? __dadd_rn(__dmul_rn(rk[k].x, res[k].x), __dmul_rn(rk[k].y, res[k].y)) : 0.0;
            }
            if (UPPER && PCG) {  // r.z (pcg.py:167), fixed pairwise order
#pragma unroll
                for (int h = 1; h < K; h <<= 1)
#pragma unroll
                    for (int k = 0; k + h < K; k += 2 * h) part[k] = __dadd_rn(part[k], part[k + h]);
                acc = __dadd_rn(acc, part[0]);
            }
            // the slot's generic accesses (mine and the solver's) before the async-proxy refill
            fence_proxy_async();
            __syncwarp();
            if (t == 0 && jw + NS < nstage) issue(jw + NS);
            WS_TRACE(1, jj, 2);
            ++jw;
        }
    }
    return acc;
}

// line warps per CTA: a 2-CTA cluster keeps 4 pairs (256 threads: the full
// register file per thread), one CTA or a 4-CTA cluster up to 8 pairs
__host__ __device__ constexpr int line_cta_warps(int C) { return C == 2 ? kLineMaxWarps / 2 : kLineMaxWarps; }

struct LineSmem {  // byte offsets into dynamic shared memory
    size_t ring_f, ring_b, bars, slots, slot_bytes, total;
};

// per CTA: two direction rings [WL][R]; per line-warp pair 4 x NS mbarriers
// (tma, full, done, rtma) and NS slots
__host__ __device__ inline LineSmem line_layout(int WL, int R, int G, int NS) {
    LineSmem m;
    m.ring_f = 0;
    m.ring_b = al128((size_t)WL * R * 8);
    m.bars = m.ring_b + al128((size_t)WL * R * 8);
    m.slots = al128(m.bars + (size_t)WL * 4 * NS * 8);
    m.slot_bytes = (size_t)G * kSlotArrays * kTileSlots * 8;
    m.total = m.slots + (size_t)WL * NS * m.slot_bytes;
    return m;
}

}  // namespace

// P^{-1} r for one system per cluster, one launch: the forward unit solve
// (with the PCG residual update in front), then y / D and the backward
// transpose solve (sparse.py:222-239, 265-275; pcg.py:142-143, 167).
//
// Warps come in pairs (line warp w: warp w of the CTA, its helper: warp
// WL + w): the line warp carries only the wavefront's dependency chain, the
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
template <bool PCG, bool SB, int G, int NS, int C>
__global__ void __launch_bounds__(64 * line_cta_warps(C), 1) ldlt_line_kernel(LineArgs a) {
    extern __shared__ __align__(128) char sm[];
    __shared__ double s_red[2][kLineMaxWarps];
    __shared__ double s_cta[2][4];
    // WL line warps (+ WL helpers) per CTA; the last CTA of a cluster may hold idle pairs
    const int W = a.warps, WL = (W + C - 1) / C, R = a.ring;
    const int warp = threadIdx.x >> 5, t = threadIdx.x & 31;
    const bool helper = warp >= WL;
    const int wl = helper ? warp - WL : warp;
    const int rank = C > 1 ? (int)cluster_rank() : 0, b = blockIdx.x / C;
    const int pw = rank * WL + wl;  // line warp = forward warp
    const bool idle = pw >= W;
    // what this system needs from this launch (uniform over the cluster)
    bool upd = false;
    if (PCG) {
        const SolveState &st = a.st;
        const int ph = st.status[b] == ST_ACTIVE ? st.phase[b] : -1;
        upd = ph == PH_ITER;
        if (!(ph == PH_ITER || ph == PH_INIT)) {
            // every thread of the cluster has read status / phase before the
            // epilogue changes them (PH_RESTART -> PH_INIT)
            if (C > 1) cluster_sync_all();
            else __syncthreads();
            if (rank == 0 && threadIdx.x == 0) bwd_epilogue(a.st, b, 0.0);  // pflag / restart bookkeeping
            return;
        }
    }
    const LineSmem m = line_layout(WL, R, G, NS);
    double *ring_f = reinterpret_cast<double *>(sm + m.ring_f);
    double *ring_b = reinterpret_cast<double *>(sm + m.ring_b);
    uint64_t *bars = reinterpret_cast<uint64_t *>(sm + m.bars) + (size_t)wl * 4 * NS;
    uint64_t *tma = bars, *full = bars + NS, *done = bars + 2 * NS, *rtma = bars + 3 * NS;
    char *slots = sm + m.slots + (size_t)wl * NS * m.slot_bytes;
    for (int i = threadIdx.x; i < WL * R; i += blockDim.x) ring_f[i] = ring_b[i] = sentinel();
    if (helper && t == 0) {
        for (int s = 0; s < 4 * NS; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    if (C > 1) cluster_sync_all();  // every ring armed before any remote write
    else __syncthreads();

    const long long vb = (long long)b * a.nslot;
    const long long db = a.d_batched ? vb : 0;
    const bool trace_on = b == 0 && rank == 0;
    const size_t fb = SB ? (size_t)b * a.fac_slots : 0;
    double acc_f = 0.0, acc_b = 0.0;
    if (!idle) {
        LineDirIO F;
        F.meta = reinterpret_cast<const int4 *>(a.meta_f);
        F.fac = a.S_f + fb;
        F.v[0] = a.in + vb;
        F.v[1] = PCG ? a.AP + vb : nullptr;
        F.nv = PCG && upd ? 2 : 1;
        F.out = a.Y + vb;
        F.rg = PCG ? a.R + vb : nullptr;
        F.ring = ring_f;
        F.w = pw;
        F.rev = false;
        F.jbase = 0;
        LineDirIO Bk;
        Bk.meta = reinterpret_cast<const int4 *>(a.meta_b);
        Bk.fac = a.S_b + fb;
        Bk.v[0] = a.Y + vb;
        Bk.v[1] = a.D + db;
        Bk.v[2] = a.rD + db;
        Bk.nv = 3;
        Bk.out = a.out + vb;
        Bk.rdot = PCG ? a.R + vb : nullptr;
        Bk.ring = ring_b;
        Bk.w = W - 1 - pw;
        Bk.rev = true;
        Bk.jbase = (F.meta[pw].y + G - 1) / G;
        if (helper) {
            const double alpha = upd ? a.st.alpha[b] : 0.0;
            acc_f = line_helper<false, PCG, G, NS>(F, t, upd, alpha, tma, full, done, rtma, slots, m.slot_bytes, wl, trace_on);
            // the backward phase reads this warp's y (and r) stores through TMA
            fence_proxy_async_global();
            __syncwarp();
            acc_b = line_helper<true, PCG, G, NS>(Bk, t, false, 0.0, tma, full, done, rtma, slots, m.slot_bytes, wl, trace_on);
        } else {
            line_solver<false, G, NS>(F, W, WL, R, wl, t, full, done, slots, m.slot_bytes, trace_on);
            line_solver<true, G, NS>(Bk, W, WL, R, wl, t, full, done, slots, m.slot_bytes, trace_on);
        }
    }
    if (PCG) {  // fixed-order reductions: lanes, helper warps, then the cluster's CTAs
        double vf = acc_f, vbk = acc_b;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            vf = __dadd_rn(vf, __shfl_down_sync(0xffffffffu, vf, off));
            vbk = __dadd_rn(vbk, __shfl_down_sync(0xffffffffu, vbk, off));
        }
        if (helper && t == 0) s_red[0][wl] = vf, s_red[1][wl] = vbk;
        __syncthreads();
        if (threadIdx.x == 0) {
            double tf = 0.0, tb = 0.0;
            for (int q = 0; q < WL; ++q) tf = __dadd_rn(tf, s_red[0][q]), tb = __dadd_rn(tb, s_red[1][q]);
            if (C > 1) {
                st_dsm(map_rank(&s_cta[0][rank], 0), tf);
                st_dsm(map_rank(&s_cta[1][rank], 0), tb);
            } else {
                fwd_epilogue(a.st, b, tf, a.drift_count);
                bwd_epilogue(a.st, b, tb);
            }
        }
    }
    if (C > 1) {  // remote rings / partials stay valid until every CTA of the cluster is done
        cluster_sync_all();
        if (PCG && rank == 0 && threadIdx.x == 0) {
            double tf = 0.0, tb = 0.0;
            for (int q = 0; q < C; ++q) tf = __dadd_rn(tf, s_cta[0][q]), tb = __dadd_rn(tb, s_cta[1][q]);
            fwd_epilogue(a.st, b, tf, a.drift_count);
            bwd_epilogue(a.st, b, tb);
        }
    }
}

int line_trace_copy(long long *out, int n) {
#ifdef NPCG_LINE_TRACE
    n = std::min(n, kTraceWarps * kTraceStages * 3);
    return (int)cudaMemcpyFromSymbol(out, g_ws_trace, n * sizeof(long long));
#else
    (void)out;
    (void)n;
    return 0;  // no timeline in this build
#endif
}

static size_t line_smem(int WL, int R, int G, int NS) { return line_layout(WL, R, G, NS).total; }

int line_config_for(const LineSched &L, int B) {
    int dev = 0, optin = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (optin <= 0) optin = 227 * 1024;
    const size_t cap = (size_t)optin - 1024;  // static shared memory
    const int W = L.fwd.warps, R = std::max(L.fwd.ring, L.bwd.ring);
    // CTAs per system: split over two SMs while the batch leaves them free;
    // more than 8 line warps always take a cluster (2 CTAs up to 16 warps,
    // 4 beyond; the last CTA may hold idle pairs)
    auto fits = [&](int c) { return (W + c - 1) / c <= line_cta_warps(c) && (c == 1 || W >= c); };
    int C = (W % 2 == 0 && 2 * B <= sms && fits(2)) ? 2 : 1;
    if (!fits(C)) C = (fits(2) && 2 * B <= sms) ? 2 : 4;
    if (const char *env = std::getenv("NPCG_LINE_CLUSTER")) {
        const int c = std::atoi(env);
        if ((c == 1 || c == 2 || c == 4) && fits(c)) C = c;
    }
    if (!fits(C)) C = fits(2) ? 2 : (fits(4) ? 4 : 0);
    if (!C) return 0;
    const int WL = (W + C - 1) / C;
    if (const char *env = std::getenv("NPCG_LINE_CFG")) {
        const int c = std::atoi(env), G = c / 16, NS = c % 16;
        if (line_shape_ok(G, NS) && line_smem(WL, R, G, NS) <= cap) return C * 256 + c;
    }
    // long stages first (the line warp's per-stage hand-offs amortise over 16
    // steps; measured 263 vs 249 systems/s against 8-step stages four deep at
    // config 2), then deeper pipelines of shorter stages
    static const int prefs[][2] = {{4, 2}, {2, 4}, {2, 3}, {1, 4}};
    for (const auto &p : prefs)
        if (line_smem(WL, R, p[0], p[1]) <= cap) return C * 256 + p[0] * 16 + p[1];
    return 0;
}

template <bool PCG, bool SB, int G, int NS, int C>
static cudaError_t launch_ldlt_t(const LineArgs &a, cudaStream_t s) {
    auto kern = ldlt_line_kernel<PCG, SB, G, NS, C>;
    const int WL = (a.warps + C - 1) / C;
    const size_t smem = line_smem(WL, a.ring, G, NS);
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    note_launch();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.B * C);
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

template <int G, int NS, int C>
static cudaError_t launch_ldlt_gc(const LineArgs &a, cudaStream_t s) {
    const bool pcg = a.mode == TRSV_PCG;
    if (pcg) return a.s_batched ? launch_ldlt_t<true, true, G, NS, C>(a, s) : launch_ldlt_t<true, false, G, NS, C>(a, s);
    return a.s_batched ? launch_ldlt_t<false, true, G, NS, C>(a, s) : launch_ldlt_t<false, false, G, NS, C>(a, s);
}

template <int C>
static cudaError_t launch_ldlt_c(const LineArgs &a, cudaStream_t s) {
    switch (a.group * 16 + a.stages) {
        case 4 * 16 + 2: return launch_ldlt_gc<4, 2, C>(a, s);
        case 2 * 16 + 4: return launch_ldlt_gc<2, 4, C>(a, s);
        case 2 * 16 + 3: return launch_ldlt_gc<2, 3, C>(a, s);
        case 1 * 16 + 4: return launch_ldlt_gc<1, 4, C>(a, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_ldlt_line(const LineArgs &a, cudaStream_t s) {
    if (!line_shape_ok(a.group, a.stages) || a.warps < 1 || (a.cluster != 1 && a.cluster != 2 && a.cluster != 4) ||
        (a.warps + a.cluster - 1) / a.cluster > line_cta_warps(a.cluster))
        return cudaErrorInvalidValue;
    switch (a.cluster) {
        case 1: return launch_ldlt_c<1>(a, s);
        case 2: return launch_ldlt_c<2>(a, s);
        default: return launch_ldlt_c<4>(a, s);
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
