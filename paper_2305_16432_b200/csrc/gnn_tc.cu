// gnn_tc.cu -- the GNN's message-passing MLPs on the 5th-generation tensor
// cores (tcgen05, sm_100a) for latent F = 64, hidden H = 64 (gnn.py:249-258
// over autodiff.py:113-137, 174-243):
//   node update  v' = MLP([v | agg]),  agg_i = sum_{p in row i} e_p * v_col(p)
//   edge update  e' = MLP([e | v_src | v_dst])
//
// fp32 accuracy from TF32 tensor cores ("3xTF32"): every fp32 operand x is
// split into x_hi = tf32(x) and x_lo = tf32(x - x_hi); a product is
// a_hi b_hi + (a_hi b_lo + a_lo b_hi), the dropped a_lo b_lo term being
// below fp32 rounding. The tensor core's own accumulation loses low bits
// (it does not round to nearest), so nothing long accumulates inside it:
// every 32-wide K chunk's big terms get a fresh TMEM accumulator, the
// correction terms one of their own, and the epilogue adds them on the
// CUDA cores in fixed order with fp32 round-to-nearest. Measured normwise
// error of the edge outputs M against the fp64 oracle at config 2: one
// tensor-core accumulator 1.4e-5, big / correction split 1.1e-5 with both
// MLPs on the tensor cores, per-chunk accumulators (this) -- see DESIGN.md;
// the FFMA tiles give 2e-6. L' parity (1e-5 normwise) is held by
// tests/test_gpu_parity.py and tests/test_gpu_fullsize.py.
//
// One persistent CTA per SM, 4 warps (128 threads; a tile is 128 rows -- edges
// or nodes: thread t owns row t in the epilogues, the gathers are
// warp-cooperative, eight lanes per row). Shared memory (1024-byte
// aligned, every operand in the canonical K-major 128-byte-swizzle layout:
// 8-row groups 1024 B apart, a row's 16-byte chunk j stored at chunk
// j ^ (row % 8)):
//   W1^T hi / lo [64 x K1]  (K1 = 192 edge / 128 node; B operand of layer 1)
//   W2^T hi / lo [64 x 64]  16 KB each  (B operand of layer 2)
//   two A buffers of one 32-wide K chunk, hi + lo [128 x 32] each (32 KB)
// Per tile: the K chunks of X ([e | v_src | v_dst], or [v | agg] with agg
// formed in CSR order by agg_rows_kernel) are gathered, split and stored while
// the previous chunk's MMAs run
// (double-buffered, completion via tcgen05.commit -> mbarrier); layer 1
// accumulates chunk c's big terms in TMEM columns [64 c, 64 c + 64) and all
// corrections in [448, 512); the epilogue sums them with b1, applies ReLU,
// splits H and stores it as layer 2's A operand (both buffers); layer 2
// accumulates in columns [0, 128) (two chunks) and [128, 192); the final
// epilogue adds b2 and writes e in place (edge) or v_out (node).
#include <cuda_runtime.h>

#include <cstdint>

#include "gnn.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

namespace npcg {

namespace {

constexpr int kTcRows = 128;            // edges per tile = UMMA M
constexpr int kTcF = 64, kTcH = 64;     // latent width, processor hidden width
template <bool NODE>
constexpr int tc_k1() { return NODE ? 2 * kTcF : 3 * kTcF; }  // layer-1 fan-in
constexpr int kAtomBytes = kTcRows * 128;  // one 32-wide K chunk of 128 rows (16 KB)
#ifndef NPCG_TC_AHEAD
#define NPCG_TC_AHEAD 2
#endif
constexpr int kTcAhead = NPCG_TC_AHEAD;  // K chunks a row's loads run ahead of the MMAs

// byte offsets in dynamic shared memory
template <bool NODE>
struct TcSmem {
    static constexpr int W1Hi = 0;
    static constexpr int W1Lo = W1Hi + kTcH * tc_k1<NODE>() * 4;
    static constexpr int W2Hi = W1Lo + kTcH * tc_k1<NODE>() * 4;
    static constexpr int W2Lo = W2Hi + kTcF * kTcH * 4;
    static constexpr int ABuf = W2Lo + kTcF * kTcH * 4;      // 2 x (hi, lo) x 16 KB
    static constexpr int Total = ABuf + 2 * 2 * kAtomBytes + 1024;  // + alignment slack
};

__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// offset of (row r, 16-byte chunk j) in a [rows x 32 fp32] swizzled K-major block
__device__ __forceinline__ uint32_t sw128(int r, int j) {
    return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((j ^ (r & 7)) << 4));
}

// smem matrix descriptor: K-major, 128-byte swizzle, 8-row groups 1024 B apart
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;            // leading byte offset (unused for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;  // stride byte offset
    d |= (uint64_t)1 << 46;            // descriptor version (sm100)
    d |= (uint64_t)2 << 61;            // SWIZZLE_128B
    return d;
}

// instruction descriptor: D fp32, A / B tf32, both K-major, M = 128, N = 64
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kTcH >> 3) << 17) |
                            ((uint32_t)(kTcRows >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(kIdesc), "r"(accum));
}

__device__ __forceinline__ void mma_commit(void *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// 16 consecutive TMEM columns of this warp's 32 lanes -> 16 registers per thread
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// store a lane's eight gathered 16-byte pieces (rows r0 + 4 i, piece j of the 32-wide K chunk)
// split hi / lo
__device__ __forceinline__ void store_split(char *hi, char *lo, int r0, int j, const float4 (&x)[8]) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int r = r0 + 4 * i;
        float4 h, l;
        h.x = tf32_rna(x[i].x), l.x = tf32_rna(x[i].x - h.x);
        h.y = tf32_rna(x[i].y), l.y = tf32_rna(x[i].y - h.y);
        h.z = tf32_rna(x[i].z), l.z = tf32_rna(x[i].z - h.z);
        h.w = tf32_rna(x[i].w), l.w = tf32_rna(x[i].w - h.w);
        *reinterpret_cast<float4 *>(hi + sw128(r, j)) = h;
        *reinterpret_cast<float4 *>(lo + sw128(r, j)) = l;
    }
}

}  // namespace

// EDGE: e <- MLP_edge([e | v_src | v_dst]); NODE: v_out <- MLP_node([v | agg]),
// for B systems (e [b][m][F], v / v_out [b][n][F]).
template <bool NODE>
__global__ void __launch_bounds__(128, 1) mp_tc_kernel(int n, long long m, int B, const int *rp, const int *src,
                                                       const int *col, const float *W1, const float *b1,
                                                       const float *W2, const float *b2, const float *ln_g,
                                                       const float *ln_b, float *e, const float *v, float *v_out,
                                                       const float *agg) {
    constexpr int kTcK1 = tc_k1<NODE>();
    using L = TcSmem<NODE>;
    constexpr int kW1Hi = L::W1Hi, kW1Lo = L::W1Lo, kW2Hi = L::W2Hi, kW2Lo = L::W2Lo, kABuf = L::ABuf;
    extern __shared__ __align__(1024) char smem_raw[];
    char *sm = reinterpret_cast<char *>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t bar[3];  // A buffer 0 / 1 consumed, layer 2 done
    __shared__ uint32_t s_tmem;
    __shared__ float sb1[kTcH], sb2[kTcF], sg[kTcF], sl[kTcF];
    const int t = threadIdx.x, warp = t >> 5;
    // weights, transposed to [out][in] (the MMA's K-major B), split hi / lo
    for (int q = t; q < kTcH * kTcK1; q += blockDim.x) {
        const int o = q / kTcK1, i = q % kTcK1;  // W1 is [in][out]
        const float w = W1[(size_t)i * kTcH + o], h = tf32_rna(w);
        const uint32_t off = (uint32_t)(i / 32) * (kTcH * 128) + (uint32_t)((o >> 3) * 1024 + (o & 7) * 128 +
                                                                          ((((i % 32) >> 2) ^ (o & 7)) << 4) + (i & 3) * 4);
        *reinterpret_cast<float *>(sm + kW1Hi + off) = h;
        *reinterpret_cast<float *>(sm + kW1Lo + off) = tf32_rna(w - h);
    }
    for (int q = t; q < kTcF * kTcH; q += blockDim.x) {
        const int o = q / kTcH, i = q % kTcH;  // W2 is [in = H][out = F]
        const float w = W2[(size_t)i * kTcF + o], h = tf32_rna(w);
        const uint32_t off = (uint32_t)(i / 32) * (kTcF * 128) + (uint32_t)((o >> 3) * 1024 + (o & 7) * 128 +
                                                                          ((((i % 32) >> 2) ^ (o & 7)) << 4) + (i & 3) * 4);
        *reinterpret_cast<float *>(sm + kW2Hi + off) = h;
        *reinterpret_cast<float *>(sm + kW2Lo + off) = tf32_rna(w - h);
    }
    for (int q = t; q < kTcH; q += blockDim.x) sb1[q] = b1[q];
    for (int q = t; q < kTcF; q += blockDim.x) {
        sb2[q] = b2[q];
        sg[q] = ln_g ? ln_g[q] : 1.f;
        sl[q] = ln_b ? ln_b[q] : 0.f;
    }
    if (t == 0) {
        for (int i = 0; i < 3; ++i) mbar_init(&bar[i], 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_proxy_async();  // weights (generic stores) -> tensor-core reads
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;
    const uint32_t tl = tmem + ((uint32_t)(warp * 32) << 16);  // this warp's TMEM lanes
    const uint32_t a_base = smem_u32(sm + kABuf);
    const uint32_t w1h = smem_u32(sm + kW1Hi), w1l = smem_u32(sm + kW1Lo);
    const uint32_t w2h = smem_u32(sm + kW2Hi), w2l = smem_u32(sm + kW2Lo);
    // A buffer u: hi at a_base + u * 2 * kAtomBytes, lo right after
    auto abuf = [&](int u, int lo) { return sm + kABuf + (u * 2 + lo) * kAtomBytes; };
    uint32_t use[2] = {0, 0}, ph2 = 0;  // completed-use counts (mbarrier parity)
    const long long items = NODE ? (long long)n : m;
    const long long tiles_per = (items + kTcRows - 1) / kTcRows, tiles = tiles_per * B;
    // Gathers are warp-cooperative: warp w stages rows 32 w .. 32 w + 31 of a tile, eight lanes
    // per row (lane l: row 4 i + l / 8 of the warp at its i-th load, 16-byte piece l % 8 of the
    // 128-byte chunk), so one load instruction fetches four complete 128-byte lines instead of
    // a 16-byte piece of 32 lines. A lane keeps its eight rows' indices, not pointers.
    const int lane = t & 31, piece = lane & 7, rsub = lane >> 3;
    struct Rows {
        int b = 0;
        long long it = 0;        // this THREAD's row (epilogue: TMEM lane = row t)
        bool live = false;
        unsigned mask = 0;       // bit i: the lane's i-th gathered row exists
        int i0[8], i1[8], i2[8];  // row index per source: e | v_src | v_dst (edge), v | agg (node)
    };
    auto setup = [&](long long tile) {
        Rows r;
        r.b = (int)(tile / tiles_per);
        const long long row0 = (tile % tiles_per) * kTcRows;
        r.live = row0 + t < items;
        r.it = r.live ? row0 + t : 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const long long item = row0 + warp * 32 + 4 * i + rsub;
            const bool ok = item < items;
            r.mask |= ok ? 1u << i : 0u;
            r.i0[i] = ok ? (int)item : 0;
            r.i1[i] = NODE ? r.i0[i] : (ok ? src[item] : 0);
            r.i2[i] = NODE ? 0 : (ok ? col[item] : 0);
        }
        return r;
    };
    // chunk c (32 consecutive features) of the lane's eight rows
    auto load_chunk = [&](const Rows &r, int c, float4 (&x)[8]) {
        const int sidx = c >> 1;
        const float *base = NODE ? (sidx == 0 ? v + ((size_t)r.b * n) * kTcF : agg + ((size_t)r.b * n) * kTcF)
                                 : (sidx == 0 ? e + ((size_t)r.b * m) * kTcF : v + ((size_t)r.b * n) * kTcF);
        const int off = (c & 1) * 32 + piece * 4;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int idx = sidx == 0 ? r.i0[i] : (sidx == 1 ? r.i1[i] : r.i2[i]);
            x[i] = (r.mask >> i) & 1u ? *reinterpret_cast<const float4 *>(base + (size_t)idx * kTcF + off)
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
    // Row loads run kTcAhead chunks ahead of the MMAs (the kernel is bound by the latency of
    // these gathers: one warp per scheduler), across tiles too: the next tile's first chunks
    // are requested before this tile's epilogues.
    constexpr int kNC = kTcK1 / 32;
    constexpr int kPre = kTcAhead < 2 ? kTcAhead : 2;  // chunks fetched across the tile boundary (plain row loads)
    float4 xq[kTcAhead + 1][8];
    Rows cur;
    if ((long long)blockIdx.x < tiles) {
        cur = setup(blockIdx.x);
#pragma unroll
        for (int c = 0; c < kPre; ++c) load_chunk(cur, c, xq[c]);
    }
    for (long long tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const int b = cur.b;
        const long long it = cur.it;
        const bool live = cur.live;
        // ---- layer 1: K chunks of 32, double-buffered A operand ----
#pragma unroll
        for (int c = kPre; c < kTcAhead && c < kNC; ++c) load_chunk(cur, c, xq[c]);
#pragma unroll
        for (int c = 0; c < kNC; ++c) {
            const int u = c & 1;
            if (c + kTcAhead < kNC) load_chunk(cur, c + kTcAhead, xq[(c + kTcAhead) % (kTcAhead + 1)]);
            if (use[u] > 0) mbar_wait(&bar[u], (use[u] - 1) & 1);  // the MMAs that last read this buffer are done
            store_split(abuf(u, 0), abuf(u, 1), warp * 32 + rsub, piece, xq[c % (kTcAhead + 1)]);
            fence_proxy_async();
            __syncthreads();
            if (t == 0) {
                tc_fence_after();
                const uint32_t ah = a_base + (uint32_t)(u * 2) * kAtomBytes, al = ah + kAtomBytes;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t ko = (uint32_t)k * 32;
                    const uint32_t bo = (uint32_t)c * (kTcH * 128) + ko;
                    mma_tf32(tmem + 64 * c, sw128_desc(ah + ko), sw128_desc(w1h + bo), k != 0);
                    mma_tf32(tmem + 448, sw128_desc(ah + ko), sw128_desc(w1l + bo), (c | k) != 0);
                    mma_tf32(tmem + 448, sw128_desc(al + ko), sw128_desc(w1h + bo), 1);
                }
                mma_commit(&bar[u]);
            }
            ++use[u];
        }
        // the next tile's first chunks: in flight during this tile's epilogues
        const long long ntile = tile + gridDim.x;
        Rows nxt;
        if (ntile < tiles) {
            nxt = setup(ntile);
#pragma unroll
            for (int c = 0; c < kPre; ++c) load_chunk(nxt, c, xq[c]);
        }
        // every layer-1 MMA done (the last commit of each buffer)
        mbar_wait(&bar[0], (use[0] - 1) & 1);
        mbar_wait(&bar[1], (use[1] - 1) & 1);
        tc_fence_after();
        // ---- epilogue 1: H = relu(X W1 + b1) -> layer 2's A operand (K = 64: both buffers) ----
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            float hv[16], hc[16];
            tmem_ld16(tl + (uint32_t)(q * 16), hv);
#pragma unroll
            for (int c = 1; c < kTcK1 / 32; ++c) {
                tmem_ld16(tl + (uint32_t)(64 * c + q * 16), hc);
#pragma unroll
                for (int i = 0; i < 16; ++i) hv[i] += hc[i];
            }
            tmem_ld16(tl + (uint32_t)(448 + q * 16), hc);
#pragma unroll
            for (int i = 0; i < 16; ++i) hv[i] += hc[i];
            float4 x[4];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                x[j] = make_float4(fmaxf(hv[4 * j] + sb1[q * 16 + 4 * j], 0.f), fmaxf(hv[4 * j + 1] + sb1[q * 16 + 4 * j + 1], 0.f),
                                   fmaxf(hv[4 * j + 2] + sb1[q * 16 + 4 * j + 2], 0.f),
                                   fmaxf(hv[4 * j + 3] + sb1[q * 16 + 4 * j + 3], 0.f));
            const int u = q >> 1;  // hidden features 0..31 -> buffer 0, 32..63 -> buffer 1
            char *hi = abuf(u, 0), *lo = abuf(u, 1);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int jj = (q & 1) * 4 + j;  // 16-byte chunk within the 32-wide row
                float4 h, l;
                h.x = tf32_rna(x[j].x), l.x = tf32_rna(x[j].x - h.x);
                h.y = tf32_rna(x[j].y), l.y = tf32_rna(x[j].y - h.y);
                h.z = tf32_rna(x[j].z), l.z = tf32_rna(x[j].z - h.z);
                h.w = tf32_rna(x[j].w), l.w = tf32_rna(x[j].w - h.w);
                *reinterpret_cast<float4 *>(hi + sw128(t, jj)) = h;
                *reinterpret_cast<float4 *>(lo + sw128(t, jj)) = l;
            }
        }
        fence_proxy_async();
        tc_fence_before();
        __syncthreads();
        if (t == 0) {
            tc_fence_after();
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int u = k >> 2;
                const uint32_t ah = a_base + (uint32_t)(u * 2) * kAtomBytes + (uint32_t)(k & 3) * 32, al = ah + kAtomBytes;
                const uint32_t bo = (uint32_t)u * (kTcF * 128) + (uint32_t)(k & 3) * 32;
                mma_tf32(tmem + 64 * u, sw128_desc(ah), sw128_desc(w2h + bo), (k & 3) != 0);
                mma_tf32(tmem + 128, sw128_desc(ah), sw128_desc(w2l + bo), k != 0);
                mma_tf32(tmem + 128, sw128_desc(al), sw128_desc(w2h + bo), 1);
            }
            mma_commit(&bar[2]);
        }
        mbar_wait(&bar[2], ph2 & 1);
        ++ph2;
        // layer 2 read both A buffers: the next tile's chunk loads wait on this too
        tc_fence_after();
        // ---- epilogue 2: e = H W2 + b2 in place | v_out = H W2 + b2 ----
        float *eo = NODE ? v_out + ((size_t)b * n + (size_t)it) * kTcF : e + ((size_t)b * m + (size_t)it) * kTcF;
        float out[kTcF];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            float ov[16], oc[16];
            tmem_ld16(tl + (uint32_t)(q * 16), ov);
            tmem_ld16(tl + (uint32_t)(64 + q * 16), oc);
#pragma unroll
            for (int i = 0; i < 16; ++i) ov[i] += oc[i];
            tmem_ld16(tl + (uint32_t)(128 + q * 16), oc);
#pragma unroll
            for (int i = 0; i < 16; ++i) out[q * 16 + i] = (ov[i] + oc[i]) + sb2[q * 16 + i];
        }
        if (ln_g) {  // north_star LayerNorm over the row (gnn.cu layer_norm_row)
            float mu = 0.f;
#pragma unroll
            for (int f = 0; f < kTcF; ++f) mu += out[f];
            mu /= (float)kTcF;
            float var = 0.f;
#pragma unroll
            for (int f = 0; f < kTcF; ++f) var = fmaf(out[f] - mu, out[f] - mu, var);
            var /= (float)kTcF;
            const float rs = 1.0f / sqrtf(var + 1e-5f);
#pragma unroll
            for (int f = 0; f < kTcF; ++f) out[f] = fmaf((out[f] - mu) * rs, sg[f], sl[f]);
        }
        if (live) {
#pragma unroll
            for (int j = 0; j < kTcF / 4; ++j)
                reinterpret_cast<float4 *>(eo)[j] = make_float4(out[4 * j], out[4 * j + 1], out[4 * j + 2], out[4 * j + 3]);
        }
        tc_fence_before();
        __syncthreads();  // TMEM reads done before the next tile's MMAs overwrite it
        cur = nxt;
    }
    tc_fence_after();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// agg[b][i][:] = sum over row i's entries p of e[b][p][:] * v[b][col p][:] (gnn.py:250-251: mul,
// segment_sum), in CSR order with one fma per term like the in-kernel form. 16 threads per
// node, a float4 each: every load is a full 256-byte row -- the gathers are coalesced and the
// kernel runs at full occupancy, which the 128-thread tensor-core kernel cannot offer them.
__global__ void __launch_bounds__(256) agg_rows_kernel(int n, long long m, int B, const int *rp, const int *col,
                                                       const float *e, const float *v, float *agg) {
    const long long total = (long long)B * n * 16;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total; q += (long long)gridDim.x * blockDim.x) {
        const long long node = q >> 4;
        const int j = (int)(q & 15), b = (int)(node / n), i = (int)(node - (long long)b * n);
        const float4 *eb = reinterpret_cast<const float4 *>(e + ((size_t)b * m) * kTcF) + j;
        const float4 *vb = reinterpret_cast<const float4 *>(v + ((size_t)b * n) * kTcF) + j;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        const int p0 = rp[i], p1 = rp[i + 1];
#pragma unroll 4
        for (int p = p0; p < p1; ++p) {
            const float4 a = eb[(size_t)p * (kTcF / 4)], x = vb[(size_t)col[p] * (kTcF / 4)];
            acc.x = fmaf(a.x, x.x, acc.x);
            acc.y = fmaf(a.y, x.y, acc.y);
            acc.z = fmaf(a.z, x.z, acc.z);
            acc.w = fmaf(a.w, x.w, acc.w);
        }
        reinterpret_cast<float4 *>(agg)[node * 16 + j] = acc;
    }
}

template <bool NODE>
static cudaError_t launch_mp_tc_t(int n, long long m, int B, const int *rp, const int *src, const int *col,
                                  const float *W1, const float *b1, const float *W2, const float *b2,
                                  const float *ln_g, const float *ln_b, float *e, const float *v, float *v_out,
                                  const float *agg, cudaStream_t s) {
    static bool configured = false;
    const int smem = TcSmem<NODE>::Total;
    if (!configured) {
        cudaError_t c = cudaFuncSetAttribute(mp_tc_kernel<NODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (c != cudaSuccess) return c;
        configured = true;
    }
    const long long items = NODE ? (long long)n : m;
    const long long tiles = (items + kTcRows - 1) / kTcRows * B;
    const int grid = (int)std::max<long long>(1, std::min<long long>(tiles, num_sms()));
    note_launch();
    mp_tc_kernel<NODE><<<grid, 128, smem, s>>>(n, m, B, rp, src, col, W1, b1, W2, b2, ln_g, ln_b, e, v, v_out, agg);
    return cudaGetLastError();
}

cudaError_t launch_mp_edge_tc(int n, long long m, int B, const int *src, const int *col, const float *W1,
                              const float *b1, const float *W2, const float *b2, const float *ln_g,
                              const float *ln_b, float *e, const float *v, cudaStream_t s) {
    return launch_mp_tc_t<false>(n, m, B, nullptr, src, col, W1, b1, W2, b2, ln_g, ln_b, e, v, nullptr, nullptr, s);
}

// agg_buf: [B][n][64] floats of scratch (the aggregated messages)
cudaError_t launch_mp_node_tc(int n, long long m, int B, const int *rp, const int *col, const float *W1,
                              const float *b1, const float *W2, const float *b2, const float *ln_g,
                              const float *ln_b, const float *e, const float *v, float *v_out, float *agg_buf,
                              cudaStream_t s) {
    if (!agg_buf) return cudaErrorInvalidValue;
    const long long total = (long long)B * n * 16;
    note_launch();
    agg_rows_kernel<<<(int)std::min<long long>((total + 255) / 256, 16LL * num_sms()), 256, 0, s>>>(n, m, B, rp, col, e, v,
                                                                                                   agg_buf);
    return launch_mp_tc_t<true>(n, m, B, rp, nullptr, col, W1, b1, W2, b2, ln_g, ln_b, const_cast<float *>(e), v,
                                v_out, agg_buf, s);
}

}  // namespace npcg
