// train.cu -- the reference's training step on the device (SURVEY.md 8(f)
// item 3): loss and parameter gradients of one (A, b, x) tuple, and Adam.
//
// Reference semantics (pcgkit, fp64 numpy + a tape):
//   * forward: gnn.forward (gnn.py:227-263), reference mode, l = l_mp = 1;
//   * symmetrize_triangulate (gnn.py:284-296);
//   * loss_data = ||(I+L') D (I+L')^T x - b||^2 through apply_learned_factor
//     (train.py:104-150), plus x0_aux_weight * ||x0hat - x||^2 when the model
//     has the x0 head (train.py:189-205);
//   * ad.backward: the rules of autodiff.py:113-253 (affine, relu, mul,
//     concat, gather_rows, segment_sum, flatten, sum_sq, sub, scale, add);
//   * adam_step (train.py:164-185).
// Everything runs in fp64 like the reference (its training tuples are small;
// B200 has full-rate fp64), with a hand-written reverse pass instead of a
// tape. Every scatter of the reference (np.add.at over edges) is a per-row
// gather here -- over the row's own entries, or through the symmetric
// pattern's pair[] for sums over incoming edges -- so results are
// deterministic; weight gradients are reduced in two fixed-order stages.
// Results differ from pcgkit's only by summation order (1e-11 relative in
// the tests). The CPU restatement is oracle/train_port.py.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "common.cuh"
#include "train.cuh"

namespace npcg {

namespace {

constexpr int kThreads = 256;

inline int grid_for(long long items) {
    return (int)std::max<long long>(1, std::min<long long>((items + kThreads - 1) / kThreads, 32LL * 1024));
}

// One input segment of an affine layer: row r reads x[(idx ? idx[r] : r) * width + k].
struct Seg {
    const double *x = nullptr;
    const int *idx = nullptr;
    int width = 0;
};
struct Segs {
    Seg s[3];
    int n = 0;
};

// Y[r][o] = b[o] + sum over the segments' columns k of X[r][k] W[k][o] (autodiff.py:113-137), optional ReLU
__global__ void __launch_bounds__(kThreads) affine_fwd_kernel(long long R, int fo, Segs in, const double *W,
                                                              const double *b, int relu, double *Y) {
    const long long total = R * fo;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long r = t / fo;
        const int o = (int)(t - r * fo);
        double acc = b[o];
        int koff = 0;
        for (int q = 0; q < in.n; ++q) {
            const Seg &sg = in.s[q];
            const double *xr = sg.x + (sg.idx ? (long long)sg.idx[r] : r) * sg.width;
            for (int k = 0; k < sg.width; ++k) acc += xr[k] * W[(size_t)(koff + k) * fo + o];
            koff += sg.width;
        }
        Y[t] = relu ? (acc > 0.0 ? acc : 0.0) : acc;
    }
}

// dX[r][k] (+)= (sum_o dY[r][o] W[koff + k][o]) * (mask ? mask[r][k] > 0 : 1): g @ W^T (autodiff.py:133)
// followed by the ReLU rule (autodiff.py:140-147) when dX is a hidden layer's gradient
__global__ void __launch_bounds__(kThreads) affine_bwd_dx_kernel(long long R, int fo, int width, int koff,
                                                                 const double *dY, const double *W,
                                                                 const double *mask, int accumulate, double *dX) {
    const long long total = R * width;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long r = t / width;
        const int k = (int)(t - r * width);
        const double *g = dY + r * fo, *w = W + (size_t)(koff + k) * fo;
        double acc = 0.0;
        for (int o = 0; o < fo; ++o) acc += g[o] * w[o];
        if (mask && !(mask[t] > 0.0)) acc = 0.0;
        dX[t] = accumulate ? dX[t] + acc : acc;
    }
}

// Weight gradient, stage 1: part[c][k][o] = sum over the rows of chunk c of X[r][k] dY[r][o]
// (x.T @ g, autodiff.py:133), with k == fi the bias row (X = 1: g.sum(axis = 0)).
// Block = (chunk, 16-row tile of W); thread (kl, ol) owns k = 16 kt + kl and columns ol + 16 j.
constexpr int kWT = 16, kRowsTile = 64, kMaxFo = 128;
__global__ void __launch_bounds__(kThreads) affine_bwd_dw_kernel(long long R, int fi, int fo, Segs in,
                                                                 const double *dY, long long chunk_rows,
                                                                 double *part) {
    __shared__ double xs[kRowsTile][kWT + 1];
    extern __shared__ double gs[];  // [kRowsTile][fo]
    const int c = blockIdx.x, kt = blockIdx.y;
    const int kl = threadIdx.x / 16, ol = threadIdx.x % 16;
    const int k = kt * kWT + kl;
    const long long r0 = c * chunk_rows, r1 = std::min<long long>(R, r0 + chunk_rows);
    double acc[kMaxFo / 16];
#pragma unroll
    for (int j = 0; j < kMaxFo / 16; ++j) acc[j] = 0.0;
    // which segment / column this thread's k reads
    int seg = -1, kk = 0;
    if (k < fi) {
        int off = 0;
        for (int q = 0; q < in.n; ++q) {
            if (k < off + in.s[q].width) {
                seg = q;
                kk = k - off;
                break;
            }
            off += in.s[q].width;
        }
    }
    for (long long rb = r0; rb < r1; rb += kRowsTile) {
        const int rows = (int)std::min<long long>(kRowsTile, r1 - rb);
        // X tile: thread (kl, ol) loads rows ol, ol + 16, ...
        for (int rr = ol; rr < kRowsTile; rr += 16) {
            double v = 0.0;
            if (rr < rows) {
                const long long r = rb + rr;
                if (k == fi) v = 1.0;
                else if (seg >= 0) {
                    const Seg &sg = in.s[seg];
                    v = sg.x[(sg.idx ? (long long)sg.idx[r] : r) * sg.width + kk];
                }
            }
            xs[rr][kl] = v;
        }
        for (int q = threadIdx.x; q < kRowsTile * fo; q += kThreads) {
            const int rr = q / fo;
            gs[q] = rr < rows ? dY[(rb + rr) * fo + (q - rr * fo)] : 0.0;
        }
        __syncthreads();
        for (int rr = 0; rr < rows; ++rr) {
            const double xv = xs[rr][kl];
#pragma unroll
            for (int j = 0; j < kMaxFo / 16; ++j)
                if (ol + 16 * j < fo) acc[j] += xv * gs[rr * fo + ol + 16 * j];
        }
        __syncthreads();
    }
    if (k <= fi) {
        double *out = part + ((size_t)c * (fi + 1) + k) * fo;
#pragma unroll
        for (int j = 0; j < kMaxFo / 16; ++j)
            if (ol + 16 * j < fo) out[ol + 16 * j] = acc[j];
    }
}

// stage 2: gW[k][o] += sum_c part[c][k][o] (c ascending); gb[o] += sum_c part[c][fi][o]
__global__ void __launch_bounds__(kThreads) affine_bwd_dw_sum_kernel(int chunks, int fi, int fo, const double *part,
                                                                     double *gW, double *gb) {
    const int total = (fi + 1) * fo;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int c = 0; c < chunks; ++c) s += part[(size_t)c * total + t];
        if (t < fi * fo) gW[t] += s;
        else gb[t - fi * fo] += s;
    }
}

// agg[i][f] = sum over row i's entries p of e[p][f] v[col[p]][f] (gnn.py:250-251: mul, segment_sum)
__global__ void __launch_bounds__(kThreads) agg_fwd_kernel(int n, int F, const int *rp, const int *col,
                                                           const double *e, const double *v, double *agg) {
    const long long total = (long long)n * F;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(t / F), f = (int)(t - (long long)i * F);
        double acc = 0.0;
        for (int p = rp[i]; p < rp[i + 1]; ++p) acc += e[(size_t)p * F + f] * v[(size_t)col[p] * F + f];
        agg[t] = acc;
    }
}

// de[p][f] += dagg[src[p]][f] v[col[p]][f]: segment_sum then mul backward (autodiff.py:177, 243)
__global__ void __launch_bounds__(kThreads) agg_bwd_e_kernel(long long m, int F, const int *src, const int *col,
                                                             const double *dagg, const double *v, double *de) {
    const long long total = m * F;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long p = t / F;
        const int f = (int)(t - p * F);
        de[t] += dagg[(size_t)src[p] * F + f] * v[(size_t)col[p] * F + f];
    }
}

// dv[j][f] += sum over edges q with dst q = j of dagg[src q][f] e[q][f] (gather_rows backward,
// autodiff.py:205-210). The pattern is symmetric: those edges are pair[p] for p in row j, and
// src(pair[p]) = col[p].
__global__ void __launch_bounds__(kThreads) agg_bwd_v_kernel(int n, int F, const int *rp, const int *col,
                                                             const int *pair, const double *dagg, const double *e,
                                                             double *dv) {
    const long long total = (long long)n * F;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int j = (int)(t / F), f = (int)(t - (long long)j * F);
        double acc = 0.0;
        for (int p = rp[j]; p < rp[j + 1]; ++p) acc += dagg[(size_t)col[p] * F + f] * e[(size_t)pair[p] * F + f];
        dv[t] += acc;
    }
}

// dv[i][f] += sum_{p in row i} (dsrc[p][f] + ddst[pair[p]][f]): backward of the two gather_rows of
// the edge MLP's input [e | v[src] | v[dst]] (gnn.py:254-257)
__global__ void __launch_bounds__(kThreads) gather_bwd_kernel(int n, int F, const int *rp, const int *pair,
                                                              const double *dsrc, const double *ddst, double *dv) {
    const long long total = (long long)n * F;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(t / F), f = (int)(t - (long long)i * F);
        double a = 0.0, b = 0.0;
        for (int p = rp[i]; p < rp[i + 1]; ++p) {
            a += dsrc[(size_t)p * F + f];
            b += ddst[(size_t)pair[p] * F + f];
        }
        dv[t] += a + b;
    }
}

// S[p] = 0.5 (M[p] + M[pair[p]]) off the diagonal, 0 on it: L' on both triangles (gnn.py:284-296)
__global__ void __launch_bounds__(kThreads) sym_kernel(long long m, const int *src, const int *col, const int *pair,
                                                       const double *M, double *S) {
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < m; p += (long long)gridDim.x * blockDim.x)
        S[p] = src[p] == col[p] ? 0.0 : 0.5 * (M[p] + M[pair[p]]);
}

// out[i] = scale[i] * (base[i] + sum over row i's entries with col > i (upper) or col < i of S[p] vec[col[p]]):
// the sweeps of apply_learned_factor (train.py:118-124) and of its backward (train.py:133-137)
__global__ void __launch_bounds__(kThreads) sweep_kernel(int n, int upper, const int *rp, const int *col,
                                                         const double *S, const double *vec, const double *base,
                                                         const double *scale, double *out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double acc = base[i];
        for (int p = rp[i]; p < rp[i + 1]; ++p) {
            const int j = col[p];
            if (upper ? j > i : j < i) acc += S[p] * vec[j];
        }
        out[i] = scale ? scale[i] * acc : acc;
    }
}

// res = y - b, gy = 2 res (sub, sum_sq: autodiff.py:160-168, 255-262); aux terms likewise
__global__ void __launch_bounds__(kThreads) residual_kernel(int n, const double *y, const double *b, double wgt,
                                                            double *res, double *g) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double r = y[i] - b[i];
        res[i] = r;
        g[i] = wgt * (2.0 * r);
    }
}

// *out (+)= wgt * sum res^2, one block, fixed order
__global__ void __launch_bounds__(1024) sumsq_kernel(int n, const double *res, double wgt, int accumulate, double *out) {
    __shared__ double red[1024];
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += 1024) s += res[i] * res[i];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int h = 512; h > 0; h >>= 1) {
        if (threadIdx.x < h) red[threadIdx.x] += red[threadIdx.x + h];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = (accumulate ? *out : 0.0) + wgt * red[0];
}

// dM[p] = 0.5 dL'(the lower slot p or pair[p] stands for), dL'_ij = g_i w_j + x_i (D t)_j (train.py:133-139)
__global__ void __launch_bounds__(kThreads) dm_kernel(long long m, const int *src, const int *col, const double *gy,
                                                      const double *w, const double *x, const double *D,
                                                      const double *t, double *dM) {
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < m; p += (long long)gridDim.x * blockDim.x) {
        int i = src[p], j = col[p];
        if (i == j) {
            dM[p] = 0.0;
            continue;
        }
        if (i < j) {
            const int s = i;
            i = j;
            j = s;
        }
        dM[p] = 0.5 * (gy[i] * w[j] + x[i] * (D[j] * t[j]));
    }
}

__global__ void __launch_bounds__(kThreads) diag_kernel(int n, const int *dp, const double *vals, double *D) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) D[i] = vals[dp[i]];
}

// train.py:164-185, one thread per parameter
__global__ void __launch_bounds__(kThreads) adam_kernel(long long count, const double *g, double gscale, double lr,
                                                        double b1, double b2, double eps, double bc1, double bc2,
                                                        double *p, double *m, double *v) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < count; q += (long long)gridDim.x * blockDim.x) {
        // numpy's operation order, unfused
        const double gr = __dmul_rn(g[q], gscale);
        double mq = m[q], vq = v[q];
        mq = __dadd_rn(mq, __dmul_rn(1.0 - b1, __dsub_rn(gr, mq)));
        vq = __dadd_rn(vq, __dmul_rn(1.0 - b2, __dsub_rn(__dmul_rn(gr, gr), vq)));
        m[q] = mq;
        v[q] = vq;
        const double num = __dmul_rn(lr, __ddiv_rn(mq, bc1));
        const double den = __dadd_rn(__dsqrt_rn(__ddiv_rn(vq, bc2)), eps);
        p[q] = __dsub_rn(p[q], __ddiv_rn(num, den));
    }
}

__global__ void __launch_bounds__(kThreads) nonfinite_kernel(long long count, const double *g, int *flag) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < count; q += (long long)gridDim.x * blockDim.x)
        if (!isfinite(g[q])) atomicOr(flag, 1);
}

}  // namespace

// ---------------------------------------------------------------------------

struct Layer {
    long long w = 0, b = 0;
    int fi = 0, fo = 0;
};

struct TrainNet::Impl {
    npcg_gnn_desc d{};
    long long count = 0;
    Layer node_enc[2], edge_enc[2], edge_dec[2], node_dec[2], mp_node[16][2], mp_edge[16][2];
    double *w = nullptr, *am = nullptr, *av = nullptr;  // weights, Adam moments
    double *ws = nullptr;                              // workspace
    size_t ws_cap = 0;
    double *part = nullptr;
    size_t part_cap = 0;
    int *flag = nullptr;
    double *loss_dev = nullptr;
};

TrainNet::TrainNet() : im(new Impl) {}
TrainNet::~TrainNet() {
    if (!im) return;
    cudaFree(im->w);
    cudaFree(im->am);
    cudaFree(im->av);
    cudaFree(im->ws);
    cudaFree(im->part);
    cudaFree(im->flag);
    cudaFree(im->loss_dev);
    delete im;
}

std::string TrainNet::init(const npcg_gnn_desc &d, const double *weights, long long n_weights) {
    if (d.l != 1 || d.l_mp != 1) return "the device training step supports l == l_mp == 1";
    if (d.north_star) return "the device training step covers the reference network (north_star mode has no reference)";
    if (d.n_mp < 1 || d.n_mp > 16) return "n_mp must be in [1, 16]";
    if (d.width < 1 || d.width > kMaxFo || d.h < 1 || d.h > kMaxFo || d.h_mp < 1 || d.h_mp > kMaxFo)
        return "layer widths must be in [1, 128]";
    Impl &m = *im;
    m.d = d;
    long long off = 0;
    auto layer = [&](Layer &L, int fi, int fo) {
        L.fi = fi;
        L.fo = fo;
        L.w = off;
        off += (long long)fi * fo;
        L.b = off;
        off += fo;
    };
    const int F = d.width;
    layer(m.node_enc[0], 1, d.h);
    layer(m.node_enc[1], d.h, F);
    layer(m.edge_enc[0], 1, d.h);
    layer(m.edge_enc[1], d.h, F);
    for (int r = 0; r < d.n_mp; ++r) {
        layer(m.mp_node[r][0], 2 * F, d.h_mp);
        layer(m.mp_node[r][1], d.h_mp, F);
        layer(m.mp_edge[r][0], 3 * F, d.h_mp);
        layer(m.mp_edge[r][1], d.h_mp, F);
    }
    layer(m.edge_dec[0], F, d.h);
    layer(m.edge_dec[1], d.h, 1);
    if (d.with_x0_head) {
        layer(m.node_dec[0], F, d.h);
        layer(m.node_dec[1], d.h, 1);
    }
    if (off != n_weights) return "weight blob length does not match the hyper-parameters";
    m.count = off;
    const size_t bytes = (size_t)std::max<long long>(off, 1) * sizeof(double);
    if (cudaMalloc(&m.w, bytes) != cudaSuccess || cudaMalloc(&m.am, bytes) != cudaSuccess ||
        cudaMalloc(&m.av, bytes) != cudaSuccess || cudaMalloc(&m.flag, sizeof(int)) != cudaSuccess ||
        cudaMalloc(&m.loss_dev, sizeof(double)) != cudaSuccess)
        return "cudaMalloc failed";
    if (cudaFuncSetAttribute(affine_bwd_dw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(kRowsTile * kMaxFo * sizeof(double))) != cudaSuccess)
        return "cudaFuncSetAttribute failed";
    cudaMemcpy(m.w, weights, (size_t)off * sizeof(double), cudaMemcpyHostToDevice);
    cudaMemset(m.am, 0, bytes);
    cudaMemset(m.av, 0, bytes);
    return "";
}

long long TrainNet::n_weights() const { return im->count; }
double *TrainNet::weights_dev() const { return im->w; }

int TrainNet::set_weights(const double *host, int reset_moments) {
    const size_t bytes = (size_t)im->count * sizeof(double);
    if (cudaMemcpy(im->w, host, bytes, cudaMemcpyHostToDevice) != cudaSuccess) return 1;
    if (reset_moments) {
        cudaMemset(im->am, 0, bytes);
        cudaMemset(im->av, 0, bytes);
    }
    return 0;
}

namespace {

struct Arena {  // bump allocator over the trainer's workspace
    double *base = nullptr;
    size_t used = 0, cap = 0;
    double *take(size_t count) {
        count = (count + 15) & ~size_t(15);
        double *p = base ? base + used : nullptr;
        used += count;
        return p;
    }
};

}  // namespace

// One tuple: forward with every activation kept, loss, reverse pass; the parameter gradient is
// ADDED to grad_accum (the caller sums tuples in index order, train.py:208-226).
int TrainNet::tuple_grad(const Pattern &A, const double *A_vals, const double *node_in, const double *edge_in,
                         const double *b, const double *x, double x0_aux_weight, double *loss_host,
                         double *grad_accum, cudaStream_t st, std::string &err) {
    Impl &M_ = *im;
    const npcg_gnn_desc &d = M_.d;
    const int n = (int)A.n, F = d.width, h = d.h, hm = d.h_mp, R = d.n_mp;
    const long long m = A.nnz;
    if (!A.symmetric || !A.full_diag) {
        err = "the training step needs a structurally symmetric pattern with a full diagonal";
        return NPCG_ERR_DATA_FORMAT;
    }
    const bool head = d.with_x0_head != 0;
    // ---- workspace: two passes over the same take() sequence (size, then pointers)
    Arena ar;
    std::vector<double *> V(R + 1), E(R + 1), AGG(R), HN(R), HE(R);
    double *h_ne, *h_ee, *h_ed, *h_nd, *Mv, *x0, *S, *D, *u, *w, *y, *res, *gy, *t, *aux, *dx0, *dM;
    double *de[2], *dv[2], *dhe, *dhn, *dsrc, *ddst, *dagg, *dhid_e, *dhid_n;
    auto layout = [&]() {
        ar.used = 0;
        for (int r = 0; r <= R; ++r) V[r] = ar.take((size_t)n * F), E[r] = ar.take((size_t)m * F);
        for (int r = 0; r < R; ++r)
            AGG[r] = ar.take((size_t)n * F), HN[r] = ar.take((size_t)n * hm), HE[r] = ar.take((size_t)m * hm);
        h_ne = ar.take((size_t)n * h), h_ee = ar.take((size_t)m * h), h_ed = ar.take((size_t)m * h);
        h_nd = ar.take((size_t)n * h);
        Mv = ar.take(m), x0 = ar.take(n), S = ar.take(m), dM = ar.take(m);
        D = ar.take(n), u = ar.take(n), w = ar.take(n), y = ar.take(n), res = ar.take(n), gy = ar.take(n);
        t = ar.take(n), aux = ar.take(n), dx0 = ar.take(n);
        for (int q = 0; q < 2; ++q) de[q] = ar.take((size_t)m * F), dv[q] = ar.take((size_t)n * F);
        dhe = ar.take((size_t)m * hm), dhn = ar.take((size_t)n * hm);
        dsrc = ar.take((size_t)m * F), ddst = ar.take((size_t)m * F), dagg = ar.take((size_t)n * F);
        dhid_e = ar.take((size_t)m * h), dhid_n = ar.take((size_t)n * h);
    };
    layout();
    if (ar.used > M_.ws_cap) {
        cudaFree(M_.ws);
        M_.ws = nullptr;
        M_.ws_cap = 0;
        if (cudaMalloc(&M_.ws, ar.used * sizeof(double)) != cudaSuccess) {
            err = "cudaMalloc failed (training workspace)";
            return NPCG_ERR_CUDA;
        }
        M_.ws_cap = ar.used;
    }
    ar.base = M_.ws;
    layout();
    // weight-gradient partials: chunks x (fi + 1) x fo for the largest layer
    const int chunks = (int)std::max<long long>(1, std::min<long long>(64, (m + 1023) / 1024));
    const size_t part_need = (size_t)chunks * (3 * F + 1) * std::max({F, h, hm});
    if (part_need > M_.part_cap) {
        cudaFree(M_.part);
        M_.part = nullptr;
        M_.part_cap = 0;
        if (cudaMalloc(&M_.part, part_need * sizeof(double)) != cudaSuccess) {
            err = "cudaMalloc failed (gradient partials)";
            return NPCG_ERR_CUDA;
        }
        M_.part_cap = part_need;
    }
    const double *Wt = M_.w;
    const int *rp = A.rp, *col = A.col, *pair = A.pair, *src = A.src;

    auto seg1 = [](const double *x, int width, const int *idx = nullptr) {
        Seg s;
        s.x = x;
        s.idx = idx;
        s.width = width;
        return s;
    };
    auto fwd = [&](long long rows, const Segs &in, const Layer &L, int relu, double *Y) {
        note_launch();
        affine_fwd_kernel<<<grid_for(rows * L.fo), kThreads, 0, st>>>(rows, L.fo, in, Wt + L.w, Wt + L.b, relu, Y);
    };
    auto one = [&](const double *x, int width) {
        Segs s;
        s.n = 1;
        s.s[0] = seg1(x, width);
        return s;
    };
    // dW / db of layer L from its input segments and dY, accumulated into grad_accum
    auto bwd_w = [&](long long rows, const Segs &in, const Layer &L, const double *dY) {
        const int ch = (int)std::max<long long>(1, std::min<long long>(chunks, (rows + 1023) / 1024));
        const long long chunk_rows = (rows + ch - 1) / ch;
        dim3 grid(ch, (L.fi + 1 + kWT - 1) / kWT);
        note_launch();
        affine_bwd_dw_kernel<<<grid, kThreads, (size_t)kRowsTile * L.fo * sizeof(double), st>>>(rows, L.fi, L.fo, in, dY,
                                                                                                 chunk_rows, M_.part);
        note_launch();
        affine_bwd_dw_sum_kernel<<<grid_for((long long)(L.fi + 1) * L.fo), kThreads, 0, st>>>(
            ch, L.fi, L.fo, M_.part, grad_accum + L.w, grad_accum + L.b);
    };
    auto bwd_x = [&](long long rows, const Layer &L, int width, int koff, const double *dY, const double *mask,
                     int accumulate, double *dX) {
        note_launch();
        affine_bwd_dx_kernel<<<grid_for(rows * width), kThreads, 0, st>>>(rows, L.fo, width, koff, dY, Wt + L.w, mask,
                                                                          accumulate, dX);
    };

    // ---- forward (gnn.py:247-263), every activation kept
    fwd(n, one(node_in, 1), M_.node_enc[0], 1, h_ne);
    fwd(n, one(h_ne, h), M_.node_enc[1], 0, V[0]);
    fwd(m, one(edge_in, 1), M_.edge_enc[0], 1, h_ee);
    fwd(m, one(h_ee, h), M_.edge_enc[1], 0, E[0]);
    std::vector<Segs> in_node(R), in_edge(R);
    for (int r = 0; r < R; ++r) {
        note_launch();
        agg_fwd_kernel<<<grid_for((long long)n * F), kThreads, 0, st>>>(n, F, rp, col, E[r], V[r], AGG[r]);
        in_node[r].n = 2;
        in_node[r].s[0] = seg1(V[r], F);
        in_node[r].s[1] = seg1(AGG[r], F);
        fwd(n, in_node[r], M_.mp_node[r][0], 1, HN[r]);
        fwd(n, one(HN[r], hm), M_.mp_node[r][1], 0, V[r + 1]);
        in_edge[r].n = 3;
        in_edge[r].s[0] = seg1(E[r], F);
        in_edge[r].s[1] = seg1(V[r + 1], F, src);
        in_edge[r].s[2] = seg1(V[r + 1], F, col);
        fwd(m, in_edge[r], M_.mp_edge[r][0], 1, HE[r]);
        fwd(m, one(HE[r], hm), M_.mp_edge[r][1], 0, E[r + 1]);
    }
    fwd(m, one(E[R], F), M_.edge_dec[0], 1, h_ed);
    fwd(m, one(h_ed, h), M_.edge_dec[1], 0, Mv);
    if (head) {
        fwd(n, one(V[R], F), M_.node_dec[0], 1, h_nd);
        fwd(n, one(h_nd, h), M_.node_dec[1], 0, x0);
    }
    // ---- loss (gnn.py:284-296, train.py:104-150)
    note_launch();
    sym_kernel<<<grid_for(m), kThreads, 0, st>>>(m, src, col, pair, Mv, S);
    note_launch();
    diag_kernel<<<grid_for(n), kThreads, 0, st>>>(n, A.dp, A_vals, D);
    note_launch();
    sweep_kernel<<<grid_for(n), kThreads, 0, st>>>(n, 1, rp, col, S, x, x, D, w);  // w = D (I+L')^T x
    note_launch();
    sweep_kernel<<<grid_for(n), kThreads, 0, st>>>(n, 0, rp, col, S, w, w, nullptr, y);  // y = (I+L') w
    note_launch();
    residual_kernel<<<grid_for(n), kThreads, 0, st>>>(n, y, b, 1.0, res, gy);
    note_launch();
    sumsq_kernel<<<1, 1024, 0, st>>>(n, res, 1.0, 0, M_.loss_dev);
    // ---- reverse pass
    note_launch();
    sweep_kernel<<<grid_for(n), kThreads, 0, st>>>(n, 1, rp, col, S, gy, gy, nullptr, t);  // t = (I+L')^T g
    note_launch();
    dm_kernel<<<grid_for(m), kThreads, 0, st>>>(m, src, col, gy, w, x, D, t, dM);
    // edge decoder
    bwd_w(m, one(h_ed, h), M_.edge_dec[1], dM);
    bwd_x(m, M_.edge_dec[1], h, 0, dM, h_ed, 0, dhid_e);
    bwd_w(m, one(E[R], F), M_.edge_dec[0], dhid_e);
    int ce = 0, cv = 0;
    bwd_x(m, M_.edge_dec[0], F, 0, dhid_e, nullptr, 0, de[ce]);
    cudaMemsetAsync(dv[cv], 0, (size_t)n * F * sizeof(double), st);
    if (head) {  // + x0_aux_weight * ||x0hat - x||^2 (train.py:201-203)
        note_launch();
        residual_kernel<<<grid_for(n), kThreads, 0, st>>>(n, x0, x, x0_aux_weight, aux, dx0);
        note_launch();
        sumsq_kernel<<<1, 1024, 0, st>>>(n, aux, x0_aux_weight, 1, M_.loss_dev);
        bwd_w(n, one(h_nd, h), M_.node_dec[1], dx0);
        bwd_x(n, M_.node_dec[1], h, 0, dx0, h_nd, 0, dhid_n);
        bwd_w(n, one(V[R], F), M_.node_dec[0], dhid_n);
        bwd_x(n, M_.node_dec[0], F, 0, dhid_n, nullptr, 1, dv[cv]);
    }
    for (int r = R - 1; r >= 0; --r) {
        // edge MLP: e' = he W1 + b1, he = relu([e | v'[src] | v'[dst]] W0 + b0)
        bwd_w(m, one(HE[r], hm), M_.mp_edge[r][1], de[ce]);
        bwd_x(m, M_.mp_edge[r][1], hm, 0, de[ce], HE[r], 0, dhe);
        bwd_w(m, in_edge[r], M_.mp_edge[r][0], dhe);
        bwd_x(m, M_.mp_edge[r][0], F, 0, dhe, nullptr, 0, de[ce ^ 1]);
        bwd_x(m, M_.mp_edge[r][0], F, F, dhe, nullptr, 0, dsrc);
        bwd_x(m, M_.mp_edge[r][0], F, 2 * F, dhe, nullptr, 0, ddst);
        note_launch();
        gather_bwd_kernel<<<grid_for((long long)n * F), kThreads, 0, st>>>(n, F, rp, pair, dsrc, ddst, dv[cv]);
        // node MLP: v' = hn W1 + b1, hn = relu([v | agg] W0 + b0)
        bwd_w(n, one(HN[r], hm), M_.mp_node[r][1], dv[cv]);
        bwd_x(n, M_.mp_node[r][1], hm, 0, dv[cv], HN[r], 0, dhn);
        bwd_w(n, in_node[r], M_.mp_node[r][0], dhn);
        bwd_x(n, M_.mp_node[r][0], F, 0, dhn, nullptr, 0, dv[cv ^ 1]);
        bwd_x(n, M_.mp_node[r][0], F, F, dhn, nullptr, 0, dagg);
        // agg = segment_sum(e * v[dst])
        note_launch();
        agg_bwd_e_kernel<<<grid_for(m * F), kThreads, 0, st>>>(m, F, src, col, dagg, V[r], de[ce ^ 1]);
        note_launch();
        agg_bwd_v_kernel<<<grid_for((long long)n * F), kThreads, 0, st>>>(n, F, rp, col, pair, dagg, E[r], dv[cv ^ 1]);
        ce ^= 1;
        cv ^= 1;
    }
    // encoders
    bwd_w(m, one(h_ee, h), M_.edge_enc[1], de[ce]);
    bwd_x(m, M_.edge_enc[1], h, 0, de[ce], h_ee, 0, dhid_e);
    bwd_w(m, one(edge_in, 1), M_.edge_enc[0], dhid_e);
    bwd_w(n, one(h_ne, h), M_.node_enc[1], dv[cv]);
    bwd_x(n, M_.node_enc[1], h, 0, dv[cv], h_ne, 0, dhid_n);
    bwd_w(n, one(node_in, 1), M_.node_enc[0], dhid_n);
    if (cudaMemcpyAsync(loss_host, M_.loss_dev, sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess || cudaGetLastError() != cudaSuccess) {
        err = "CUDA failure in the training step";
        return NPCG_ERR_CUDA;
    }
    return NPCG_OK;
}

// adam_step (train.py:164-185) with g = grad * grad_scale; returns NPCG_ERR_INVALID_FACTOR-like
// nonfinite = 1 (NonFiniteGradientError) without touching the weights
int TrainNet::adam(const double *grad, double grad_scale, long long t, double lr, double b1, double b2, double eps,
                   int *nonfinite, cudaStream_t st) {
    Impl &m = *im;
    cudaMemsetAsync(m.flag, 0, sizeof(int), st);
    note_launch();
    nonfinite_kernel<<<grid_for(m.count), kThreads, 0, st>>>(m.count, grad, m.flag);
    int f = 0;
    if (cudaMemcpyAsync(&f, m.flag, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return NPCG_ERR_CUDA;
    *nonfinite = f;
    if (f) return NPCG_OK;
    const double bc1 = 1.0 - std::pow(b1, (double)t), bc2 = 1.0 - std::pow(b2, (double)t);
    note_launch();
    adam_kernel<<<grid_for(m.count), kThreads, 0, st>>>(m.count, grad, grad_scale, lr, b1, b2, eps, bc1, bc2, m.w, m.am,
                                                        m.av);
    return cudaGetLastError() == cudaSuccess ? NPCG_OK : NPCG_ERR_CUDA;
}

}  // namespace npcg
