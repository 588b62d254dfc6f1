// trsv.cuh -- launch interface of the level-pipelined triangular solves.
#pragma once
#include "common.cuh"
#include "pattern.h"

namespace npcg {

constexpr int kTrsvThreads = 256;
constexpr int kTrsvPD = 4;  // pipeline depth in levels (struct 2*PD ahead, vectors PD ahead)

enum TrsvMode : int { TRSV_PLAIN = 0, TRSV_PCG = 1 };
enum TrsvOp : int { TOP_SKIP = 0, TOP_SOLVE = 1, TOP_UPDATE = 2, TOP_RESET = 3 };

// Unsolved marker for triangular-solve outputs (a NaN payload arithmetic
// never produces); consumers poll until the value differs from it.
constexpr unsigned long long kSentinel = 0xFFF4BADC0FFEE000ull;

struct TrsvArgs {
    int n = 0, B = 1, G = 1, groups = 1, units = 0;
    int upper = 0, mode = TRSV_PLAIN;
    Schedule sched{};
    const double *S = nullptr;  // factor values, packed in this direction's level order
    int s_batched = 0;          // S laid out [group][padded entries][G]
    const double *D = nullptr;
    int d_batched = 0;
    double *in = nullptr;   // forward: r ; backward: y (re-armed after use in PCG mode)
    double *out = nullptr;  // forward: y ; backward: z (must start as sentinels)
    double *R = nullptr, *X = nullptr;
    const double *P = nullptr, *AP = nullptr;
    SolveState st{};
    double *partial = nullptr;
    Ctl *ctl = nullptr;
    int *drift_count = nullptr;
};

// Shared-memory layout (bytes) of one CTA.
struct TrsvSmem {
    unsigned ring_off = 0, lvl_off = 0, mbar_off = 0, struct_off = 0, data_off = 0, total = 0;
    int lvl_n = 0, struct_bytes = 0, sval_off = 0, data_bytes = 0, ext_off = 0, slab = 0;
};

TrsvSmem trsv_smem_plan(const Schedule &S, int G, int s_batched);

// Line-wavefront P^{-1} (trsv_line.cu): one cluster of 1, 2 or 4 CTAs per
// system, one lane per grid line; ONE launch runs the forward solve, the
// diagonal scaling and the backward solve (ldlt_line_kernel). Every vector
// is in line order, system-major: element (slot q, system b) at b*nslot + q.
struct LineArgs {
    int B = 1, mode = TRSV_PLAIN;
    int cluster = 1, group = 2, stages = 2;  // CTAs per cluster, tiles per pipeline stage, stages per warp
    int kr = 1;  // systems per cluster (1, 2 or 4; more than one needs a shared factor and B % kr == 0)
    int nslot = 0, warps = 0, ring = 64;     // ring: steps per warp's incoming value ring (LineDir::ring)
    const int *meta_f = nullptr, *meta_b = nullptr;  // LineDir::meta of the two directions
    long long fac_slots = 0;
    const double *S_f = nullptr, *S_b = nullptr;  // packed factor values ([b][fac_slots] when s_batched)
    int s_batched = 0;
    // diag(A) and its correctly rounded reciprocal in line order ([nslot] or
    // [b][nslot], padding 1.0): y / D is formed exactly from them
    const double *D = nullptr, *rD = nullptr;
    int d_batched = 0;
    const double *in = nullptr;   // forward right-hand side (PCG: r_k)
    double *Y = nullptr;          // forward result y (scratch between the phases)
    double *out = nullptr;        // z
    double *R = nullptr;          // PCG: r_{k+1} = r_k - alpha Ap, written by the forward phase
    const double *AP = nullptr;   // PCG: A p
    SolveState st{};
    int *drift_count = nullptr;
    long long *trace = nullptr;  // debug timeline buffer (set by launch_ldlt_line)
};
// ---- launch geometry shared by trsv_line.cu and the kernel instances ----
// operand stages per warp (a slot is refilled the stage after its use): three
// up to 3-tile stages, two for 4-tile stages (shared memory)
// (tiles per stage, stages in flight) combinations the kernel is built for
__host__ __device__ constexpr bool line_shape_ok(int G, int NS) {
    return (G == 4 && NS == 2) || (G == 3 && NS == 3) || (G == 2 && (NS == 3 || NS == 4)) || (G == 1 && NS == 4);
}

__host__ __device__ inline size_t al128(size_t x) { return (x + 127) & ~size_t(127); }
__host__ __device__ constexpr int slot_arrays(int KR) { return kLineKinds + 3 * KR; }  // arrays of a stage slot
constexpr int kLineMaxKR = 4;
// line warps per CTA: a 2-CTA cluster keeps 4 pairs (256 threads: the full
// register file per thread), one CTA or a 4-CTA cluster up to 8 pairs
__host__ __device__ constexpr int line_cta_warps(int C) { return C == 2 ? kLineMaxWarps / 2 : kLineMaxWarps; }
struct LineSmem {  // byte offsets into dynamic shared memory
    size_t ring_f, ring_b, bars, slots, slot_bytes, total;
};

// per CTA: two direction rings [WL][R][KR]; per line-warp pair 4 x NS mbarriers
// (tma, full, done, rtma) and NS slots
__host__ __device__ inline LineSmem line_layout(int WL, int R, int G, int NS, int KR) {
    LineSmem m;
    m.ring_f = 0;
    m.ring_b = al128((size_t)WL * R * KR * 8);
    m.bars = m.ring_b + al128((size_t)WL * R * KR * 8);
    m.slots = al128(m.bars + (size_t)WL * 4 * NS * 8);
    m.slot_bytes = (size_t)G * slot_arrays(KR) * kTileSlots * 8;
    m.total = m.slots + (size_t)WL * NS * m.slot_bytes;
    return m;
}
inline size_t line_smem_bytes(int WL, int R, int G, int NS, int KR) { return line_layout(WL, R, G, NS, KR).total; }
constexpr int kLineTraceWarps = 4 * 8, kLineTraceStages = 1024;  // debug timeline (NPCG_LINE_TRACE builds)
// Launch shape (kr << 16 | cluster * 256 + group * 16 + stages) for B systems,
// kr of them per cluster, that fits shared memory; 0 when none does.
// NPCG_LINE_CFG (group * 16 + stages) and NPCG_LINE_CLUSTER override.
int line_config_for(const LineSched &L, int B, int KR = 1);
inline int line_cfg_cluster(int cfg) { return (cfg >> 8) & 0xff; }
int line_trace_copy(long long *out, int n);  // debug timeline (NPCG_LINE_TRACE builds)
cudaError_t launch_ldlt_line(const LineArgs &a, cudaStream_t s);
// the instances behind it: k<systems per cluster><p: PCG mode, n: plain> (trsv_line_k*.cu)
cudaError_t launch_ldlt_k1p(const LineArgs &a, cudaStream_t s);
cudaError_t launch_ldlt_k1n(const LineArgs &a, cudaStream_t s);
cudaError_t launch_ldlt_k2p(const LineArgs &a, cudaStream_t s);
cudaError_t launch_ldlt_k2n(const LineArgs &a, cudaStream_t s);
cudaError_t launch_ldlt_k4p(const LineArgs &a, cudaStream_t s);
cudaError_t launch_ldlt_k4n(const LineArgs &a, cudaStream_t s);
// rD[q] = 1 / D[q] (correctly rounded), count entries
cudaError_t launch_reciprocal(long long count, const double *D, double *rD, cudaStream_t s);
// factor values S[p * ps + b * bs] -> line order of `L` (per system when batched)
void launch_line_factor_pack(const LineDir &L, int B, int sb, long long ps, long long bs, const double *S,
                             double *packed, cudaStream_t s);
// Level-synchronous solve (trsv_level.cu): one cooperative launch per
// direction, a grid barrier per level; vectors RHS-minor (i * B + b),
// factor values packed in the direction's entry order ([e][B] when batched).
struct LevelSyncArgs {
    int B = 1, upper = 0, mode = TRSV_PLAIN, grid = 0;
    int nlev = 0;
    const int *lvl_ptr = nullptr, *rows = nullptr, *eptr = nullptr, *ecol = nullptr;
    const double *S = nullptr;
    int s_batched = 0;
    const double *D = nullptr;  // diag(A) [i * B + b] or [i]
    int d_batched = 0;
    const double *in = nullptr;  // forward: r ; backward: y
    double *out = nullptr;       // forward: y ; backward: z
    double *R = nullptr;         // PCG: r (forward writes r_{k+1}, backward reads it for r.z)
    const double *AP = nullptr;
    SolveState st{};
    double *partial = nullptr;   // [grid][B]
    unsigned *bar = nullptr;     // [2] zero-initialised barrier words
    int *drift_count = nullptr;
    // dependency-flag mode (no barrier between levels): flags[row * nflag +
    // f] >= epoch once row's column group f is final in this launch;
    // zero-initialised, epoch strictly increasing across launches
    unsigned *flags = nullptr;
    unsigned epoch = 0;
    int max_rows = 0;   // widest level (flag-mode grid sizing)
    int sleep_ns = 20;  // flag poll back-off
};
// flag words per row: one per warp of 32 columns (B % 32 == 0), else one per column
inline int level_flag_groups(int B) { return B % 32 == 0 ? B / 32 : B; }
int level_sync_grid(int B);
cudaError_t launch_level_sync(const LevelSyncArgs &a, cudaStream_t s);
// packed[e * B + b] = S[perm[e] * B + b] (batched) | packed[e] = S[perm[e]]
void launch_level_factor_pack(long long entries, int B, int sb, const int *perm, const double *S, double *packed,
                              cudaStream_t s);
cudaError_t launch_trsv(const TrsvArgs &a, cudaStream_t s);
// factor values (CSR order, symmetric S) -> packed level order of `sched`
void launch_factor_pack(const Schedule &sched, int B, int G, int s_batched, const double *S, double *packed,
                        cudaStream_t s);
void launch_fill_sentinel(long long count, double *p, cudaStream_t s);

}  // namespace npcg
