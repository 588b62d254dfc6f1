// gnn.cu -- sm_100a kernels for the learned preconditioner's GNN
// (reference: pkg/src/pcgkit/gnn.py:227-318 over autodiff.py:113-253).
//
// Reference-mode network, fp32 arithmetic (north_star: "fp32 GNN"), input
// statistics and all factor assembly in fp64:
//   v = MLP_node_enc((b - mu_b)/sd_b)          e = MLP_edge_enc((A - mu_A)/sd_A)
//   repeat n_mp: agg_i = sum_{p in row i} e_p * v_{col p}
//                v = MLP_mp.node([v | agg]);  e = MLP_mp.edge([e | v_src | v_dst])
//   M = MLP_edge_dec(e);  L'_s = (M_s + M_pair(s)) / 2;  D = diag(A)
// The per-round MLPs run as register-tiled fp32 GEMM tiles from shared
// memory inside persistent CTAs (weights loaded once per CTA); the
// encoders / decoders are one thread per item with weights broadcast
// from shared memory. Nothing is atomically accumulated: aggregation is a
// CSR row walk in stored order, so the pass is deterministic.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "gnn.cuh"
#include "kernels.cuh"

namespace npcg {

constexpr int kGnnThreads = 256;
constexpr int kMaxHidden = 128;

GnnDev::~GnnDev() {
    if (w) cudaFree(w);
}

std::string gnn_init(GnnDev &g, const npcg_gnn_desc &d, const double *weights, int64_t n_weights) {
    if (d.l != 1 || d.l_mp != 1) return "GPU GNN supports l == l_mp == 1 (one hidden layer per MLP)";
    if (d.width != 16 && d.width != 64) return "latent width must be 16 or 64";
    if (d.n_mp < 1 || d.n_mp > 16) return "n_mp must be in [1, 16]";
    if (d.h < 1 || d.h > kMaxHidden) return "encoder/decoder hidden width must be in [1, 128]";
    const int F = d.width, hm = d.h_mp;
    const bool ok_hm = (F == 16 && (hm == 8 || hm == 16 || hm == 32)) || (F == 64 && (hm == 32 || hm == 64));
    if (!ok_hm) return "unsupported (width, h_mp) combination";
    g.d = d;
    int64_t off = 0;
    auto layer = [&](LayerOff &L, int fi, int fo) {
        L.w = off;
        off += (int64_t)fi * fo;
        L.b = off;
        off += fo;
    };
    if (d.north_star && d.dim != 2 && d.dim != 3) return "north_star mode needs dim 2 or 3";
    const int node_in = d.north_star ? 2 : 1, edge_in = d.north_star ? 2 + d.dim : 1;
    layer(g.node_enc[0], node_in, d.h);
    layer(g.node_enc[1], d.h, F);
    layer(g.edge_enc[0], edge_in, d.h);
    layer(g.edge_enc[1], d.h, F);
    for (int r = 0; r < d.n_mp; ++r) {
        layer(g.mp_node[r][0], 2 * F, hm);
        layer(g.mp_node[r][1], hm, F);
        layer(g.mp_edge[r][0], 3 * F, hm);
        layer(g.mp_edge[r][1], hm, F);
    }
    layer(g.edge_dec[0], F, d.h);
    layer(g.edge_dec[1], d.h, 1);
    if (d.with_x0_head) {
        layer(g.node_dec[0], F, d.h);
        layer(g.node_dec[1], d.h, 1);
    }
    if (d.north_star) {  // LayerNorm gain / shift per stack, after every layer
        layer(g.ln_node_enc, 1, F);
        layer(g.ln_edge_enc, 1, F);
        for (int r = 0; r < d.n_mp; ++r) {
            layer(g.ln_mp_node[r], 1, F);
            layer(g.ln_mp_edge[r], 1, F);
        }
    }
    if (off != n_weights) return "weight blob length does not match the hyper-parameters";
    std::vector<float> h(off);
    for (int64_t i = 0; i < off; ++i) h[i] = (float)weights[i];
    if (cudaMalloc(&g.w, std::max<int64_t>(off, 1) * sizeof(float)) != cudaSuccess) return "cudaMalloc failed";
    if (cudaMemcpy(g.w, h.data(), off * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess)
        return "cudaMemcpy failed";
    g.n_floats = off;
    return "";
}

// ---------------------------------------------------------------------------
// per-column mean / population std (gnn.py:42-51), fp64, fixed order
// ---------------------------------------------------------------------------
__global__ void colstat_partial_kernel(long long count, int B, const double *x, const double *mean,
                                       double *partial) {
    __shared__ double red[kGnnThreads];
    const int cols = B < kGnnThreads ? B : kGnnThreads;
    const int rows_per = kGnnThreads / cols;
    for (int b0 = 0; b0 < B; b0 += cols) {
        const int b = b0 + threadIdx.x % cols, r0 = threadIdx.x / cols;
        double s = 0.0;
        if (b < B && r0 < rows_per) {
            const double mu = mean ? mean[b] : 0.0;
            for (long long i = (long long)blockIdx.x * rows_per + r0; i < count; i += (long long)gridDim.x * rows_per) {
                const double v = x[(size_t)i * B + b];
                s = mean ? __dadd_rn(s, __dmul_rn(v - mu, v - mu)) : __dadd_rn(s, v);
            }
        }
        red[threadIdx.x] = s;
        __syncthreads();
        if (threadIdx.x < cols && b0 + threadIdx.x < B) {
            double t = 0.0;
            for (int q = 0; q < rows_per; ++q) t = __dadd_rn(t, red[q * cols + threadIdx.x]);
            partial[(size_t)blockIdx.x * B + b0 + threadIdx.x] = t;
        }
        __syncthreads();
    }
}

// mode 0: out = sum/count (mean); mode 1: out = sqrt(sum/count) or 1 if 0.
__global__ void colstat_final_kernel(long long count, int B, int nblk, const double *partial, double *out,
                                     int mode) {
    for (int b = threadIdx.x; b < B; b += blockDim.x) {
        double t = 0.0;
        for (int k = 0; k < nblk; ++k) t = __dadd_rn(t, partial[(size_t)k * B + b]);
        if (count == 0) {
            out[b] = mode ? 1.0 : 0.0;
            continue;
        }
        const double m = t / (double)count;
        if (mode == 0) out[b] = m;
        else {
            const double sd = sqrt(m);
            out[b] = sd > 0.0 ? sd : 1.0;
        }
    }
}

// ---------------------------------------------------------------------------
// LayerNorm over a row of F features (north_star): population variance,
// eps 1e-5, then gain and shift (oracle/port.py _layer_norm)
// ---------------------------------------------------------------------------
constexpr float kLnEps = 1e-5f;

template <int F>
__device__ __forceinline__ void layer_norm_row(float (&x)[F], const float *g, const float *b) {
    float mu = 0.f;
#pragma unroll
    for (int f = 0; f < F; ++f) mu += x[f];
    mu /= (float)F;
    float var = 0.f;
#pragma unroll
    for (int f = 0; f < F; ++f) var = fmaf(x[f] - mu, x[f] - mu, var);
    var /= (float)F;
    const float rs = 1.0f / sqrtf(var + kLnEps);
#pragma unroll
    for (int f = 0; f < F; ++f) x[f] = fmaf((x[f] - mu) * rs, g[f], b[f]);
}

// in-place LayerNorm of rows [rows][F] (the FFMA processor path)
template <int F>
__global__ void __launch_bounds__(kGnnThreads) ln_rows_kernel(long long rows, float *x, const float *g,
                                                              const float *b) {
    __shared__ float sg[F], sb[F];
    for (int q = threadIdx.x; q < F; q += blockDim.x) sg[q] = g[q], sb[q] = b[q];
    __syncthreads();
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows; r += (long long)gridDim.x * blockDim.x) {
        float v[F];
        float4 *p = reinterpret_cast<float4 *>(x + (size_t)r * F);
#pragma unroll
        for (int f4 = 0; f4 < F / 4; ++f4) {
            const float4 t = p[f4];
            v[4 * f4] = t.x, v[4 * f4 + 1] = t.y, v[4 * f4 + 2] = t.z, v[4 * f4 + 3] = t.w;
        }
        layer_norm_row<F>(v, sg, sb);
#pragma unroll
        for (int f4 = 0; f4 < F / 4; ++f4) p[f4] = make_float4(v[4 * f4], v[4 * f4 + 1], v[4 * f4 + 2], v[4 * f4 + 3]);
    }
}

// ---------------------------------------------------------------------------
// encoders: WIN inputs -> h -> F  (gnn.py:247-248; north_star: more inputs
// and a LayerNorm). Items are (system b, index i); input feature k of item
// i is x[k][i*B + b] (batched) or x[k][i] (shared), standardised with its
// per-system statistics; out[(b*count + i)*F]
// ---------------------------------------------------------------------------
constexpr int kMaxEncIn = 5;
struct EncIn {
    const double *x[kMaxEncIn];
    int xb[kMaxEncIn];
    const double *mean[kMaxEncIn], *sd[kMaxEncIn];  // [B] each
};

template <int F, int WIN>
__global__ void __launch_bounds__(kGnnThreads) encode_kernel(long long count, int B, EncIn in, int normalize,
                                                             const float *W1, const float *b1, const float *W2,
                                                             const float *b2, int h, const float *ln_g,
                                                             const float *ln_b, float *out) {
    __shared__ float sW1[WIN * kMaxHidden], sb1[kMaxHidden];
    __shared__ __align__(16) float sW2[kMaxHidden * F];
    __shared__ __align__(16) float sb2[F];
    __shared__ float sg[F], sb[F];
    for (int k = threadIdx.x; k < WIN * h; k += blockDim.x) sW1[k] = W1[k];
    for (int k = threadIdx.x; k < h; k += blockDim.x) sb1[k] = b1[k];
    for (int k = threadIdx.x; k < h * F; k += blockDim.x) sW2[k] = W2[k];
    for (int k = threadIdx.x; k < F; k += blockDim.x) {
        sb2[k] = b2[k];
        sg[k] = ln_g ? ln_g[k] : 1.f;
        sb[k] = ln_b ? ln_b[k] : 0.f;
    }
    __syncthreads();
    // two rows per thread: every weight read from shared memory feeds two rows' FMAs (the
    // broadcast loads are what the one-row form waits on)
    constexpr int R = 2;
    const long long total = count * B, pairs = (total + R - 1) / R;
    for (long long qp = blockIdx.x * (long long)blockDim.x + threadIdx.x; qp < pairs;
         qp += (long long)gridDim.x * blockDim.x) {
        float xf[R][WIN];
        bool on[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const long long q = qp * R + r;
            on[r] = q < total;
            const long long qq = on[r] ? q : 0;
            const int b = (int)(qq / count);
            const long long i = qq % count;
#pragma unroll
            for (int k = 0; k < WIN; ++k) {
                double xv = in.xb[k] ? in.x[k][(size_t)i * B + b] : in.x[k][i];
                if (normalize) xv = (xv - in.mean[k][b]) / in.sd[k][b];
                xf[r][k] = (float)xv;
            }
        }
        float acc[R][F];
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int f = 0; f < F; ++f) acc[r][f] = sb2[f];
        for (int k = 0; k < h; ++k) {
            float hk[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                float a = sb1[k];
#pragma unroll
                for (int c = 0; c < WIN; ++c) a = fmaf(xf[r][c], sW1[c * h + k], a);
                hk[r] = fmaxf(a, 0.0f);
            }
            const float4 *w4 = reinterpret_cast<const float4 *>(sW2 + k * F);
#pragma unroll
            for (int f4 = 0; f4 < F / 4; ++f4) {
                const float4 w = w4[f4];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    acc[r][4 * f4 + 0] = fmaf(hk[r], w.x, acc[r][4 * f4 + 0]);
                    acc[r][4 * f4 + 1] = fmaf(hk[r], w.y, acc[r][4 * f4 + 1]);
                    acc[r][4 * f4 + 2] = fmaf(hk[r], w.z, acc[r][4 * f4 + 2]);
                    acc[r][4 * f4 + 3] = fmaf(hk[r], w.w, acc[r][4 * f4 + 3]);
                }
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (!on[r]) continue;
            const long long q = qp * R + r;
            const int b = (int)(q / count);
            const long long i = q % count;
            if (ln_g) layer_norm_row<F>(acc[r], sg, sb);
            float4 *o4 = reinterpret_cast<float4 *>(out + ((size_t)b * count + i) * F);
#pragma unroll
            for (int f4 = 0; f4 < F / 4; ++f4)
                o4[f4] = make_float4(acc[r][4 * f4], acc[r][4 * f4 + 1], acc[r][4 * f4 + 2], acc[r][4 * f4 + 3]);
        }
    }
}

// north_star edge geometry: geo[k][p] = pos[col p][k] - pos[src p][k] (k < dim), geo[dim][p] = |d|
__global__ void edge_geometry_kernel(long long m, int dim, const int *src, const int *col, const double *pos,
                                     double *geo) {
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < m; p += (long long)gridDim.x * blockDim.x) {
        const int i = src[p], j = col[p];
        double s2 = 0.0;
        for (int k = 0; k < dim; ++k) {
            const double d = pos[(size_t)j * dim + k] - pos[(size_t)i * dim + k];
            geo[(size_t)k * m + p] = d;
            s2 = fma(d, d, s2);
        }
        geo[(size_t)dim * m + p] = sqrt(s2);
    }
}

// ---------------------------------------------------------------------------
// register-tiled  OUT[TE][N] = act(XT^T[TE][K] . W[K][N] + b[N])  from smem
// XT is K x (TE+PAD) (transposed input), W is K x N.
// ---------------------------------------------------------------------------
template <int TE, int N>
struct TileShape {
    static constexpr int PER = TE * N / kGnnThreads;
    static constexpr int TN = PER >= 4 ? 4 : PER;
    static constexpr int TM = PER / TN;
    static constexpr int COLG = N / TN;  // column groups
    static_assert(TE * N % kGnnThreads == 0, "tile must cover the block");
    static_assert(COLG * (TE / TM) == kGnnThreads, "tile shape");
};

constexpr int kPad = 4;

template <int TE, int K, int N, bool RELU>
__device__ __forceinline__ void tile_gemm(const float *XT, const float *W, const float *bias,
                                          float (&acc)[TileShape<TE, N>::TM][TileShape<TE, N>::TN]) {
    using S = TileShape<TE, N>;
    const int cx = threadIdx.x % S::COLG, ry = threadIdx.x / S::COLG;
    const int n0 = cx * S::TN, m0 = ry * S::TM;
#pragma unroll
    for (int a = 0; a < S::TM; ++a)
#pragma unroll
        for (int c = 0; c < S::TN; ++c) acc[a][c] = bias[n0 + c];
#pragma unroll 4
    for (int k = 0; k < K; ++k) {
        float xv[S::TM], wv[S::TN];
#pragma unroll
        for (int a = 0; a < S::TM; ++a) xv[a] = XT[k * (TE + kPad) + m0 + a];
        if constexpr (S::TN == 4) {
            const float4 w = *reinterpret_cast<const float4 *>(W + k * N + n0);
            wv[0] = w.x;
            wv[1] = w.y;
            wv[2] = w.z;
            wv[3] = w.w;
        } else {
#pragma unroll
            for (int c = 0; c < S::TN; ++c) wv[c] = W[k * N + n0 + c];
        }
#pragma unroll
        for (int a = 0; a < S::TM; ++a)
#pragma unroll
            for (int c = 0; c < S::TN; ++c) acc[a][c] = fmaf(xv[a], wv[c], acc[a][c]);
    }
    if (RELU) {
#pragma unroll
        for (int a = 0; a < S::TM; ++a)
#pragma unroll
            for (int c = 0; c < S::TN; ++c) acc[a][c] = fmaxf(acc[a][c], 0.0f);
    }
}

// One message-passing half-round. NODE: in = [v | agg] (K = 2F), out -> v_out.
// EDGE: in = [e | v_src | v_dst] (K = 3F), out -> e (in place).
template <int F, int H, int TE, bool NODE>
__global__ void __launch_bounds__(kGnnThreads) mp_kernel(int n, long long m, int B, const int *rp,
                                                         const int *col, const int *src, const float *W1,
                                                         const float *b1, const float *W2, const float *b2,
                                                         float *e, const float *v, float *v_out) {
    constexpr int K1 = NODE ? 2 * F : 3 * F;
    extern __shared__ __align__(16) float smem[];
    float *sW1 = smem;                  // K1 x H
    float *sW2 = sW1 + K1 * H;          // H x F
    float *sb1 = sW2 + H * F;           // H
    float *sb2 = sb1 + H;               // F
    float *XT = sb2 + F;                // K1 x (TE+PAD)
    float *HT = XT + K1 * (TE + kPad);  // H x (TE+PAD)
    for (int q = threadIdx.x; q < K1 * H; q += blockDim.x) sW1[q] = W1[q];
    for (int q = threadIdx.x; q < H * F; q += blockDim.x) sW2[q] = W2[q];
    for (int q = threadIdx.x; q < H; q += blockDim.x) sb1[q] = b1[q];
    for (int q = threadIdx.x; q < F; q += blockDim.x) sb2[q] = b2[q];
    const long long items = NODE ? (long long)n : m;
    const long long tiles_per = (items + TE - 1) / TE;
    const long long tiles = tiles_per * B;
    using S1 = TileShape<TE, H>;
    using S2 = TileShape<TE, F>;
    for (long long tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const int b = (int)(tile / tiles_per);
        const long long base = (tile % tiles_per) * TE;
        const float *eb = e + (size_t)b * m * F;
        const float *vb = v + (size_t)b * n * F;
        __syncthreads();  // previous tile done with XT / HT (and weights loaded)
        // gather the input tile, transposed: XT[c][t]
        for (int q = threadIdx.x; q < TE * K1; q += blockDim.x) {
            const int t = q / K1, c = q % K1;
            const long long it = base + t;
            float val = 0.0f;
            if (it < items) {
                if (NODE) {
                    if (c < F) {
                        val = vb[(size_t)it * F + c];
                    } else {  // agg_i = sum_p e_p * v_col(p), CSR order (autodiff.py:221-243)
                        const int f = c - F;
                        float s = 0.0f;
                        for (int p = rp[it]; p < rp[it + 1]; ++p)
                            s = fmaf(eb[(size_t)p * F + f], vb[(size_t)col[p] * F + f], s);
                        val = s;
                    }
                } else {
                    if (c < F) val = eb[(size_t)it * F + c];
                    else if (c < 2 * F) val = vb[(size_t)src[it] * F + (c - F)];
                    else val = vb[(size_t)col[it] * F + (c - 2 * F)];
                }
            }
            XT[c * (TE + kPad) + t] = val;
        }
        __syncthreads();
        {
            float acc[S1::TM][S1::TN];
            tile_gemm<TE, K1, H, true>(XT, sW1, sb1, acc);
            const int cx = threadIdx.x % S1::COLG, ry = threadIdx.x / S1::COLG;
#pragma unroll
            for (int a = 0; a < S1::TM; ++a)
#pragma unroll
                for (int c = 0; c < S1::TN; ++c) HT[(cx * S1::TN + c) * (TE + kPad) + ry * S1::TM + a] = acc[a][c];
        }
        __syncthreads();
        {
            float acc[S2::TM][S2::TN];
            tile_gemm<TE, H, F, false>(HT, sW2, sb2, acc);
            const int cx = threadIdx.x % S2::COLG, ry = threadIdx.x / S2::COLG;
            float *outb = NODE ? v_out + (size_t)b * n * F : e + (size_t)b * m * F;
#pragma unroll
            for (int a = 0; a < S2::TM; ++a) {
                const long long it = base + ry * S2::TM + a;
                if (it >= items) continue;
                float *o = outb + (size_t)it * F + cx * S2::TN;
                if constexpr (S2::TN == 4) {
                    *reinterpret_cast<float4 *>(o) = make_float4(acc[a][0], acc[a][1], acc[a][2], acc[a][3]);
                } else {
#pragma unroll
                    for (int c = 0; c < S2::TN; ++c) o[c] = acc[a][c];
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// decoders: F -> h -> 1 (gnn.py:259-262); out[i*B + b] (vector layout), fp64
// ---------------------------------------------------------------------------
template <int F>
__global__ void __launch_bounds__(kGnnThreads) decode_kernel(long long count, int B, const float *x,
                                                             const float *W1, const float *b1, const float *W2,
                                                             const float *b2, int h, double *out) {
    __shared__ __align__(16) float sW1T[kMaxHidden * F];  // [h][F]
    __shared__ float sb1[kMaxHidden], sW2[kMaxHidden];
    for (int q = threadIdx.x; q < h * F; q += blockDim.x) {
        const int k = q / F, c = q % F;
        sW1T[q] = W1[c * h + k];
    }
    for (int k = threadIdx.x; k < h; k += blockDim.x) {
        sb1[k] = b1[k];
        sW2[k] = W2[k];
    }
    __syncthreads();
    const float bout = b2[0];
    constexpr int R = 2;  // rows per thread (see encode_kernel)
    const long long total = count * B, pairs = (total + R - 1) / R;
    for (long long qp = blockIdx.x * (long long)blockDim.x + threadIdx.x; qp < pairs;
         qp += (long long)gridDim.x * blockDim.x) {
        float xr[R][F];
        bool on[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const long long q = qp * R + r;
            on[r] = q < total;
            const long long qq = on[r] ? q : 0;
            const int b = (int)(qq / count);
            const long long i = qq % count;
            const float4 *x4 = reinterpret_cast<const float4 *>(x + ((size_t)b * count + i) * F);
#pragma unroll
            for (int f4 = 0; f4 < F / 4; ++f4) {
                const float4 t = x4[f4];
                xr[r][4 * f4] = t.x;
                xr[r][4 * f4 + 1] = t.y;
                xr[r][4 * f4 + 2] = t.z;
                xr[r][4 * f4 + 3] = t.w;
            }
        }
        float o[R];
#pragma unroll
        for (int r = 0; r < R; ++r) o[r] = bout;
        for (int k = 0; k < h; ++k) {
            float a[R];
#pragma unroll
            for (int r = 0; r < R; ++r) a[r] = sb1[k];
            const float4 *w4 = reinterpret_cast<const float4 *>(sW1T + k * F);
#pragma unroll
            for (int f4 = 0; f4 < F / 4; ++f4) {
                const float4 w = w4[f4];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    a[r] = fmaf(xr[r][4 * f4], w.x, a[r]);
                    a[r] = fmaf(xr[r][4 * f4 + 1], w.y, a[r]);
                    a[r] = fmaf(xr[r][4 * f4 + 2], w.z, a[r]);
                    a[r] = fmaf(xr[r][4 * f4 + 3], w.w, a[r]);
                }
            }
#pragma unroll
            for (int r = 0; r < R; ++r) o[r] = fmaf(fmaxf(a[r], 0.0f), sW2[k], o[r]);
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (!on[r]) continue;
            const long long q = qp * R + r;
            const int b = (int)(q / count);
            const long long i = q % count;
            out[(size_t)i * B + b] = (double)o[r];
        }
    }
}

// L'_s = 0.5 (M_s + M_pair(s)) on every off-diagonal slot (gnn.py:284-296);
// S is symmetric by construction since fp addition commutes.
__global__ void symm_kernel(long long nnz, int B, const int *pair, const int *src, const int *col, const double *M,
                            double *S, int *nonfinite) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < nnz * B;
         q += (long long)gridDim.x * blockDim.x) {
        const long long p = q / B;
        const int b = (int)(q % B);
        double s = 0.0;
        if (src[p] != col[p]) {
            s = 0.5 * (M[q] + M[(size_t)pair[p] * B + b]);
            if (!isfinite(s)) *nonfinite = 1;
        }
        S[q] = s;
    }
}

// D = diag(A) (gnn.py:301-304); records the first row with d <= 0 and
// non-finite diagonals (LowerFactor validation, sparse.py:189-190).
__global__ void diag_kernel(int n, int B, const int *dp, const double *A, int ab, double *D, int *bad_row,
                            int *nonfinite) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < (long long)n * B;
         q += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(q / B), b = (int)(q % B);
        const double d = ab ? A[(size_t)dp[i] * B + b] : A[dp[i]];
        D[q] = d;
        if (d <= 0.0) atomicMin(bad_row, i);
        if (!isfinite(d)) *nonfinite = 1;
    }
}

// tcgen05 edge update (gnn_tc.cu), F = H = 64; NPCG_GNN_TC=0 keeps the FFMA tiles
cudaError_t launch_mp_edge_tc(int n, long long m, int B, const int *src, const int *col, const float *W1,
                              const float *b1, const float *W2, const float *b2, const float *ln_g,
                              const float *ln_b, float *e, const float *v, cudaStream_t s);
cudaError_t launch_mp_node_tc(int n, long long m, int B, const int *rp, const int *col, const float *W1,
                              const float *b1, const float *W2, const float *b2, const float *ln_g,
                              const float *ln_b, const float *e, const float *v, float *v_out, float *agg_buf,
                              cudaStream_t s);
static bool gnn_tc_enabled() {
    static int on = -1;
    if (on < 0) {
        const char *env = std::getenv("NPCG_GNN_TC");
        on = env ? std::atoi(env) != 0 : 1;
    }
    return on != 0;
}

// north_star factor P = L L^T with L_ii = exp(M_ii), L_ij = (M_ij + M_ji) / 2
// (i > j), in the solver's unit-lower form: S_p = L_ij / L_jj on both slots of
// the pair, D_i = L_ii^2 (oracle/port.py assemble_exp).
__global__ void exp_diag_kernel(int n, int B, const int *dp, const double *M, double *D, double *d, int *nonfinite) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < (long long)n * B;
         q += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(q / B), b = (int)(q % B);
        const double li = exp(M[(size_t)dp[i] * B + b]);
        d[q] = li;
        D[q] = li * li;
        if (!(isfinite(li) && li > 0.0 && isfinite(li * li))) *nonfinite = 1;
    }
}

__global__ void exp_factor_kernel(long long nnz, int B, const int *pair, const int *src, const int *col,
                                  const double *M, const double *d, double *S, int *nonfinite) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < nnz * B;
         q += (long long)gridDim.x * blockDim.x) {
        const long long p = q / B;
        const int b = (int)(q % B);
        double s = 0.0;
        const int r = src[p], c = col[p];
        if (r != c) {
            const double l = 0.5 * (M[q] + M[(size_t)pair[p] * B + b]);
            s = l / d[(size_t)(r < c ? r : c) * B + b];
            if (!isfinite(s)) *nonfinite = 1;
        }
        S[q] = s;
    }
}

// ---------------------------------------------------------------------------
template <int F, int H, int TE>
static cudaError_t run_rounds(const GnnDev &g, const Pattern &A, int B, float *aggbuf, float *e, float *v, float *v2,
                              float **v_final, cudaStream_t s) {
    const int n = (int)A.n;
    const long long m = A.nnz;
    const size_t smem_node = sizeof(float) * ((2 * F) * H + H * F + H + F + (2 * F) * (TE + kPad) + H * (TE + kPad));
    const size_t smem_edge = sizeof(float) * ((3 * F) * H + H * F + H + F + (3 * F) * (TE + kPad) + H * (TE + kPad));
    cudaFuncSetAttribute(mp_kernel<F, H, TE, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_node);
    cudaFuncSetAttribute(mp_kernel<F, H, TE, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_edge);
    int occ_n = 1, occ_e = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_n, mp_kernel<F, H, TE, true>, kGnnThreads, smem_node);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_e, mp_kernel<F, H, TE, false>, kGnnThreads, smem_edge);
    const long long tn = ((long long)n + TE - 1) / TE * B, te = (m + TE - 1) / TE * B;
    const int gn = (int)std::max<long long>(1, std::min<long long>(tn, (long long)std::max(occ_n, 1) * num_sms()));
    const int ge = (int)std::max<long long>(1, std::min<long long>(te, (long long)std::max(occ_e, 1) * num_sms()));
    const bool tc = F == 64 && H == 64 && gnn_tc_enabled();
    const bool ln = g.d.north_star != 0;
    const float *w = g.w;
    auto ln_rows = [&](long long rows, float *x, const LayerOff &L) {
        if (!ln || tc) return cudaSuccess;  // the tensor-core kernels normalise in their epilogue
        const int grid = (int)std::max<long long>(1, std::min<long long>((rows + kGnnThreads - 1) / kGnnThreads, 8 * num_sms()));
        note_launch();
        ln_rows_kernel<F><<<grid, kGnnThreads, 0, s>>>(rows, x, w + L.w, w + L.b);
        return cudaGetLastError();
    };
    for (int r = 0; r < g.d.n_mp; ++r) {
        const float *lng_n = ln ? w + g.ln_mp_node[r].w : nullptr, *lnb_n = ln ? w + g.ln_mp_node[r].b : nullptr;
        const float *lng_e = ln ? w + g.ln_mp_edge[r].w : nullptr, *lnb_e = ln ? w + g.ln_mp_edge[r].b : nullptr;
        if (tc) {
            cudaError_t c = launch_mp_node_tc(n, m, B, A.rp, A.col, w + g.mp_node[r][0].w, w + g.mp_node[r][0].b,
                                              w + g.mp_node[r][1].w, w + g.mp_node[r][1].b, lng_n, lnb_n, e, v, v2,
                                              aggbuf, s);
            if (c != cudaSuccess) return c;
        } else {
            note_launch(); mp_kernel<F, H, TE, true><<<gn, kGnnThreads, smem_node, s>>>(
                n, m, B, A.rp, A.col, A.src, w + g.mp_node[r][0].w, w + g.mp_node[r][0].b, w + g.mp_node[r][1].w,
                w + g.mp_node[r][1].b, e, v, v2);
            if (cudaError_t c = ln_rows((long long)n * B, v2, g.ln_mp_node[r])) return c;
        }
        std::swap(v, v2);
        if (tc) {
            cudaError_t c = launch_mp_edge_tc(n, m, B, A.src, A.col, w + g.mp_edge[r][0].w, w + g.mp_edge[r][0].b,
                                              w + g.mp_edge[r][1].w, w + g.mp_edge[r][1].b, lng_e, lnb_e, e, v, s);
            if (c != cudaSuccess) return c;
            continue;
        }
        note_launch(); mp_kernel<F, H, TE, false><<<ge, kGnnThreads, smem_edge, s>>>(
            n, m, B, A.rp, A.col, A.src, w + g.mp_edge[r][0].w, w + g.mp_edge[r][0].b, w + g.mp_edge[r][1].w,
            w + g.mp_edge[r][1].b, e, v, nullptr);
        if (cudaError_t c = ln_rows(m * B, e, g.ln_mp_edge[r])) return c;
    }
    *v_final = v;
    return cudaGetLastError();
}

template <int F>
static cudaError_t encode(const GnnDev &g, long long count, int B, int win, const EncIn &in, const LayerOff *L,
                          const LayerOff *ln, float *out, cudaStream_t s) {
    const long long total = count * B;
    const int grid = (int)std::max<long long>(1, std::min<long long>((total + kGnnThreads - 1) / kGnnThreads, 8 * num_sms()));
    const float *w = g.w;
    const float *lg = ln ? w + ln->w : nullptr, *lb = ln ? w + ln->b : nullptr;
    note_launch();
    switch (win) {
        case 1: encode_kernel<F, 1><<<grid, kGnnThreads, 0, s>>>(count, B, in, g.d.normalize, w + L[0].w, w + L[0].b, w + L[1].w, w + L[1].b, g.d.h, lg, lb, out); break;
        case 2: encode_kernel<F, 2><<<grid, kGnnThreads, 0, s>>>(count, B, in, g.d.normalize, w + L[0].w, w + L[0].b, w + L[1].w, w + L[1].b, g.d.h, lg, lb, out); break;
        case 4: encode_kernel<F, 4><<<grid, kGnnThreads, 0, s>>>(count, B, in, g.d.normalize, w + L[0].w, w + L[0].b, w + L[1].w, w + L[1].b, g.d.h, lg, lb, out); break;
        case 5: encode_kernel<F, 5><<<grid, kGnnThreads, 0, s>>>(count, B, in, g.d.normalize, w + L[0].w, w + L[0].b, w + L[1].w, w + L[1].b, g.d.h, lg, lb, out); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

template <int F>
static cudaError_t decode(const GnnDev &g, long long count, int B, const float *x, const LayerOff *L, double *out,
                          cudaStream_t s) {
    const long long total = count * B;
    const int grid = (int)std::max<long long>(1, std::min<long long>((total + kGnnThreads - 1) / kGnnThreads, 8 * num_sms()));
    note_launch(); decode_kernel<F><<<grid, kGnnThreads, 0, s>>>(count, B, x, g.w + L[0].w, g.w + L[0].b, g.w + L[1].w,
                                                   g.w + L[1].b, g.d.h, out);
    return cudaGetLastError();
}

static cudaError_t stats(long long count, int B, const double *x, double *mean, double *sd, double *partial,
                         cudaStream_t s) {
    const int nblk = (int)std::max<long long>(1, std::min<long long>((count + 1023) / 1024, 2 * num_sms()));
    note_launch(); colstat_partial_kernel<<<nblk, kGnnThreads, 0, s>>>(count, B, x, nullptr, partial);
    note_launch(); colstat_final_kernel<<<1, kGnnThreads, 0, s>>>(count, B, nblk, partial, mean, 0);
    note_launch(); colstat_partial_kernel<<<nblk, kGnnThreads, 0, s>>>(count, B, x, mean, partial);
    note_launch(); colstat_final_kernel<<<1, kGnnThreads, 0, s>>>(count, B, nblk, partial, sd, 1);
    return cudaGetLastError();
}

template <int F>
static int build_F(const GnnDev &g, const Pattern &A, int B, const double *A_vals, int ab, const double *rhs,
                   double *S, double *D, double *edge_out, double *x0_out, int64_t *pivot, cudaStream_t s,
                   std::string &err, const GnnMesh *mesh) {
    const bool ns = g.d.north_star != 0;
    if (ns && (!mesh || !mesh->pos || !mesh->boundary)) {
        err = "north_star mode needs the mesh (positions, boundary flags)";
        return NPCG_ERR_ARGUMENT;
    }
    const int n = (int)A.n;
    const long long m = A.nnz;
    float *e = nullptr, *v = nullptr, *v2 = nullptr;
    double *M = nullptr, *st = nullptr;
    int *flags = nullptr;
    float *vfin = nullptr;
    const int Bs = ab ? B : 1;  // systems with distinct A values
    auto ck = [&](cudaError_t c) {
        if (c != cudaSuccess && err.empty()) err = cudaGetErrorString(c);
        return c == cudaSuccess;
    };
    keep_pool_memory();
    bool ok = ck(cudaMallocAsync((void **)&e, sizeof(float) * std::max<long long>(m * F * B, 1), s)) &&
              ck(cudaMallocAsync((void **)&v, sizeof(float) * std::max<long long>((long long)n * F * B, 1), s)) &&
              ck(cudaMallocAsync((void **)&v2, sizeof(float) * std::max<long long>((long long)n * F * B, 1), s)) &&
              ck(cudaMallocAsync((void **)&M, sizeof(double) * std::max<long long>(m * B, 1), s)) &&
              ck(cudaMallocAsync((void **)&st, sizeof(double) * (16 * B + 2 * num_sms() * (size_t)B + 8), s)) &&
              ck(cudaMallocAsync((void **)&flags, sizeof(int) * 4, s));
    // tensor-core path: the aggregated messages of a round, formed by their own full-occupancy
    // kernel (gnn_tc.cu agg_rows_kernel)
    float *aggbuf = nullptr;
    if (ok && F == 64 && g.d.h_mp == 64 && gnn_tc_enabled())
        ok = ck(cudaMallocAsync((void **)&aggbuf, sizeof(float) * std::max<long long>((long long)n * F * B, 1), s));
    double *geo = nullptr, *dl = nullptr;  // north_star: edge geometry [dim+1][m], diag(L) [n][B]
    if (ok && ns)
        ok = ck(cudaMallocAsync((void **)&geo, sizeof(double) * std::max<long long>((long long)(g.d.dim + 1) * m, 1), s)) &&
             ck(cudaMallocAsync((void **)&dl, sizeof(double) * std::max<long long>((long long)n * B, 1), s));
    int h_flags[4] = {n, 0, 0, 0};  // bad_row, nonfinite diag, nonfinite L'
    if (ok) {
        // per-system mean / sd of every input feature: slots [k][B] in st
        double *partial = st + 16 * B;
        auto mean_of = [&](int k) { return st + (size_t)(2 * k) * B; };
        auto sd_of = [&](int k) { return st + (size_t)(2 * k + 1) * B; };
        ok = ck(cudaMemcpyAsync(flags, h_flags, sizeof(h_flags), cudaMemcpyHostToDevice, s));
        // feature k: (data, batched, count) -> statistics slot k (gnn.py:42-51, 239-245)
        auto feature_stats = [&](int k, const double *x, int xb, long long count) {
            if (!ok || !g.d.normalize) return;
            const int cols = xb ? B : 1;
            ok = ck(stats(count, cols, x, mean_of(k), sd_of(k), partial, s));
            for (int b = 1; b < B && ok && !xb; ++b)  // shared feature: broadcast to every system
                ok = ck(cudaMemcpyAsync(mean_of(k) + b, mean_of(k), 8, cudaMemcpyDeviceToDevice, s)) &&
                     ck(cudaMemcpyAsync(sd_of(k) + b, sd_of(k), 8, cudaMemcpyDeviceToDevice, s));
        };
        EncIn nin{}, ein{};
        int nwin = 1, ewin = 1;
        nin.x[0] = rhs, nin.xb[0] = 1;
        ein.x[0] = A_vals, ein.xb[0] = ab;
        feature_stats(0, rhs, 1, n);
        feature_stats(1, A_vals, ab, m);
        nin.mean[0] = mean_of(0), nin.sd[0] = sd_of(0);
        ein.mean[0] = mean_of(1), ein.sd[0] = sd_of(1);
        if (ok && ns) {  // (b, boundary flag); (A, d_1..d_dim, |d|), d = pos[dst] - pos[src]
            const int dim = g.d.dim;
            note_launch();
            edge_geometry_kernel<<<(int)std::min<long long>((m + 255) / 256, 8 * num_sms()), 256, 0, s>>>(
                m, dim, A.src, A.col, mesh->pos, geo);
            ok = ck(cudaGetLastError());
            nwin = 2;
            nin.x[1] = mesh->boundary, nin.xb[1] = 0;
            feature_stats(2, mesh->boundary, 0, n);
            nin.mean[1] = mean_of(2), nin.sd[1] = sd_of(2);
            ewin = 2 + dim;
            for (int k = 0; k <= dim; ++k) {
                ein.x[1 + k] = geo + (size_t)k * m, ein.xb[1 + k] = 0;
                feature_stats(3 + k, geo + (size_t)k * m, 0, m);
                ein.mean[1 + k] = mean_of(3 + k), ein.sd[1 + k] = sd_of(3 + k);
            }
        }
        if (ok) ok = ck(encode<F>(g, n, B, nwin, nin, g.node_enc, ns ? &g.ln_node_enc : nullptr, v, s));
        if (ok) ok = ck(encode<F>(g, m, B, ewin, ein, g.edge_enc, ns ? &g.ln_edge_enc : nullptr, e, s));
        if (ok) {
            const int hm = g.d.h_mp;
            cudaError_t c = cudaErrorInvalidValue;
            if (F == 16 && hm == 16) c = run_rounds<16, 16, 64>(g, A, B, aggbuf, e, v, v2, &vfin, s);
            else if (F == 16 && hm == 8) c = run_rounds<16, 8, 64>(g, A, B, aggbuf, e, v, v2, &vfin, s);
            else if (F == 16 && hm == 32) c = run_rounds<16, 32, 64>(g, A, B, aggbuf, e, v, v2, &vfin, s);
            else if (F == 64 && hm == 64) c = run_rounds<64, 64, 32>(g, A, B, aggbuf, e, v, v2, &vfin, s);
            else if (F == 64 && hm == 32) c = run_rounds<64, 32, 32>(g, A, B, aggbuf, e, v, v2, &vfin, s);
            ok = ck(c);
        }
        double *Mout = edge_out ? edge_out : M;
        if (ok) ok = ck(decode<F>(g, m, B, e, g.edge_dec, Mout, s));
        if (ok && x0_out && g.d.with_x0_head) ok = ck(decode<F>(g, n, B, vfin, g.node_dec, x0_out, s));
        if (ok && !ns) {
            const int grid = (int)std::min<long long>((m * B + 255) / 256 + 1, 8192);
            note_launch(); symm_kernel<<<grid, 256, 0, s>>>(m, B, A.pair, A.src, A.col, Mout, S, flags + 2);
            note_launch(); diag_kernel<<<(int)std::min<long long>(((long long)n * B + 255) / 256 + 1, 8192), 256, 0, s>>>(
                n, B, A.dp, A_vals, ab, D, flags, flags + 1);
            ok = ck(cudaGetLastError());
        } else if (ok) {  // P = L L^T, exp on the diagonal
            note_launch(); exp_diag_kernel<<<(int)std::min<long long>(((long long)n * B + 255) / 256 + 1, 8192), 256, 0, s>>>(
                n, B, A.dp, Mout, D, dl, flags + 1);
            const int grid = (int)std::min<long long>((m * B + 255) / 256 + 1, 8192);
            note_launch(); exp_factor_kernel<<<grid, 256, 0, s>>>(m, B, A.pair, A.src, A.col, Mout, dl, S, flags + 2);
            ok = ck(cudaGetLastError());
        }
        if (ok) ok = ck(cudaMemcpyAsync(h_flags, flags, sizeof(h_flags), cudaMemcpyDeviceToHost, s)) &&
                     ck(cudaStreamSynchronize(s));
    }
    cudaFreeAsync(e, s);
    cudaFreeAsync(v, s);
    cudaFreeAsync(v2, s);
    cudaFreeAsync(M, s);
    cudaFreeAsync(st, s);
    cudaFreeAsync(flags, s);
    if (aggbuf) cudaFreeAsync(aggbuf, s);
    if (geo) cudaFreeAsync(geo, s);
    if (dl) cudaFreeAsync(dl, s);
    if (!ok) return NPCG_ERR_CUDA;
    if (h_flags[0] < n) {
        *pivot = h_flags[0];
        err = "nonpositive diagonal entry at row " + std::to_string(h_flags[0]);
        return NPCG_ERR_NOT_SPD;
    }
    if (h_flags[1]) {
        err = "diagonal must be finite and strictly positive";
        return NPCG_ERR_INVALID_FACTOR;
    }
    if (h_flags[2]) {
        err = "factor values must be finite";
        return NPCG_ERR_INVALID_FACTOR;
    }
    return NPCG_OK;
}

int gnn_build(const GnnDev &g, const Pattern &A, int B, const double *A_vals, int ab, const double *rhs, double *S,
              double *D, double *edge_out, double *x0_out, int64_t *pivot, cudaStream_t s, std::string &err,
              const GnnMesh *mesh) {
    if (g.d.width == 16) return build_F<16>(g, A, B, A_vals, ab, rhs, S, D, edge_out, x0_out, pivot, s, err, mesh);
    return build_F<64>(g, A, B, A_vals, ab, rhs, S, D, edge_out, x0_out, pivot, s, err, mesh);
}

}  // namespace npcg
