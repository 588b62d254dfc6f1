// fem.cu -- P1 triangle / tetrahedron FEM assembly into a fixed CSR pattern,
// on the device (the input side of the solve path).
//
// Reference semantics: pkg/src/pcgkit/fem.py:42-69 (element_stiffness /
// element_mass per triangle) and fem.py:116-134 (COO triplets in element
// order, rows = repeat(tri, 3), cols = tile(tri, 3), summed by
// SparseMatrixCsr.from_coo after a stable (row, col) lexsort). The host mirror
// is paper_2305_16432_b200/inputs.py (element_blocks, Assembler), which the
// tests pin bitwise to pcgkit.fem. Tetrahedra (configs 4 / 5; pcgkit is 2-D
// only) follow inputs.tet_blocks operation for operation: K_ij = |T| grad l_i .
// grad l_j from the edge cross products, M_ij = |T| (1 + d_ij) / 20.
//
// Layout: the plan keeps, per CSR slot, the run [starts[p], starts[p+1]) of
// triplet ids (e * NV^2 + NV i + j, block entry (i, j) of element e; NV = 3
// or 4 vertices per element) in lexsort
// order. One thread owns one (slot, system) pair -- system index fastest, so a
// warp reads one coefficient row / vertex pair for all its systems -- and
// recomputes each contributing element entry from the vertices with the
// reference's operation order (unfused fp64), so no (nt, 3, 3) block array is
// ever written. A slot's run is summed exactly like numpy's add.reduceat:
// first element + pairwise_sum(rest) (sequential from -0.0 below 8 terms, eight
// interleaved accumulators up to 128).
#include <cuda_runtime.h>

#include <algorithm>
#include <numeric>
#include <vector>

#include "common.cuh"
#include "fem.cuh"

namespace npcg {

namespace {

constexpr double kMassDiag = 2.0 / 12.0, kMassOff = 1.0 / 12.0;  // fem.py mass template / 12

template <int NV>
struct Elem;

template <>
struct Elem<3> {  // one triangle's geometry, fem.py:42-69 operation order
    double bs[3], cs[3], twice_abs;
    bool bad;
};

template <>
struct Elem<4> {  // one tetrahedron: gradients of the hat functions and the volume (inputs.tet_blocks)
    double g[4][3], vol;
    bool bad;
};

template <int NV>
__device__ __forceinline__ Elem<NV> element(const int *tri, const double *V, int vb, int B, int b, int e);

template <>
__device__ __forceinline__ Elem<3> element<3>(const int *tri, const double *V, int vb, int B, int b, int e) {
    double x[3], y[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const long long v = tri[3 * (long long)e + k];
        x[k] = V[(v * 2 + 0) * vb + (vb > 1 ? b : 0)];
        y[k] = V[(v * 2 + 1) * vb + (vb > 1 ? b : 0)];
    }
    Elem<3> E;
    const double twice = __dsub_rn(__dmul_rn(__dsub_rn(x[1], x[0]), __dsub_rn(y[2], y[0])),
                                   __dmul_rn(__dsub_rn(y[1], y[0]), __dsub_rn(x[2], x[0])));
    E.bad = !(twice > 0.0);
    E.twice_abs = fabs(twice);
    E.bs[0] = __dsub_rn(y[1], y[2]);
    E.bs[1] = __dsub_rn(y[2], y[0]);
    E.bs[2] = __dsub_rn(y[0], y[1]);
    E.cs[0] = __dsub_rn(x[2], x[1]);
    E.cs[1] = __dsub_rn(x[0], x[2]);
    E.cs[2] = __dsub_rn(x[1], x[0]);
    return E;
}

// numpy.cross of two 3-vectors: each component one product minus another, unfused
__device__ __forceinline__ void cross3(const double (&a)[3], const double (&b)[3], double (&c)[3]) {
    c[0] = __dsub_rn(__dmul_rn(a[1], b[2]), __dmul_rn(a[2], b[1]));
    c[1] = __dsub_rn(__dmul_rn(a[2], b[0]), __dmul_rn(a[0], b[2]));
    c[2] = __dsub_rn(__dmul_rn(a[0], b[1]), __dmul_rn(a[1], b[0]));
}

template <>
__device__ __forceinline__ Elem<4> element<4>(const int *tet, const double *V, int vb, int B, int b, int e) {
    double p[4][3];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const long long v = tet[4 * (long long)e + k];
#pragma unroll
        for (int d = 0; d < 3; ++d) p[k][d] = V[(v * 3 + d) * vb + (vb > 1 ? b : 0)];
    }
    double e1[3], e2[3], e3[3], c23[3], c31[3], c12[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        e1[d] = __dsub_rn(p[1][d], p[0][d]);
        e2[d] = __dsub_rn(p[2][d], p[0][d]);
        e3[d] = __dsub_rn(p[3][d], p[0][d]);
    }
    cross3(e2, e3, c23);
    cross3(e3, e1, c31);
    cross3(e1, e2, c12);
    const double det = __dadd_rn(__dadd_rn(__dmul_rn(e1[0], c23[0]), __dmul_rn(e1[1], c23[1])), __dmul_rn(e1[2], c23[2]));
    Elem<4> E;
    E.bad = !(det > 0.0);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        E.g[1][d] = __ddiv_rn(c23[d], det);
        E.g[2][d] = __ddiv_rn(c31[d], det);
        E.g[3][d] = __ddiv_rn(c12[d], det);
        E.g[0][d] = -__dadd_rn(__dadd_rn(E.g[1][d], E.g[2][d]), E.g[3][d]);
    }
    E.vol = __ddiv_rn(det, 6.0);
    return E;
}

// entry (i, j) of the (coefficient-scaled) stiffness or of the mass block
template <bool MASS>
__device__ __forceinline__ double entry(const Elem<3> &E, int i, int j, double c, bool scaled) {
    if (MASS) return __dmul_rn(__ddiv_rn(E.twice_abs, 2.0), i == j ? kMassDiag : kMassOff);
    const double k = __ddiv_rn(__dadd_rn(__dmul_rn(E.bs[i], E.bs[j]), __dmul_rn(E.cs[i], E.cs[j])),
                               __dmul_rn(2.0, E.twice_abs));
    return scaled ? __dmul_rn(k, c) : k;  // K * c[:, None, None]
}

template <bool MASS>
__device__ __forceinline__ double entry(const Elem<4> &E, int i, int j, double c, bool scaled) {
    if (MASS) return __dmul_rn(__ddiv_rn(E.vol, 20.0), i == j ? 2.0 : 1.0);
    double gi[3], gj[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {  // register-resident selects instead of dynamic indexing
        gi[d] = i == 0 ? E.g[0][d] : i == 1 ? E.g[1][d] : i == 2 ? E.g[2][d] : E.g[3][d];
        gj[d] = j == 0 ? E.g[0][d] : j == 1 ? E.g[1][d] : j == 2 ? E.g[2][d] : E.g[3][d];
    }
    const double dots = __dadd_rn(__dadd_rn(__dmul_rn(gi[0], gj[0]), __dmul_rn(gi[1], gj[1])), __dmul_rn(gi[2], gj[2]));
    const double k = __dmul_rn(E.vol, dots);
    return scaled ? __dmul_rn(k, c) : k;
}

// numpy add.reduceat of term(q0) .. term(q1 - 1): a[0] + pairwise_sum(a[1:])
// (numpy umath loops_utils.h: below 8 terms a sequential sum from -0.0, which
// keeps signed zeros; up to 128 terms eight interleaved accumulators)
template <class F>
__device__ __forceinline__ double reduceat_run(int q0, int q1, F term) {
    const double first = term(q0);
    const int n = q1 - q0 - 1;
    double rest;
    if (n < 8) {
        rest = -0.0;
        for (int q = q0 + 1; q < q1; ++q) rest = __dadd_rn(rest, term(q));
    } else {  // n <= 128 (checked when the plan is built)
        double r[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) r[k] = term(q0 + 1 + k);
        int i = 8;
        for (; i < n - (n % 8); i += 8)
#pragma unroll
            for (int k = 0; k < 8; ++k) r[k] = __dadd_rn(r[k], term(q0 + 1 + i + k));
        rest = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < n; ++i) rest = __dadd_rn(rest, term(q0 + 1 + i));
    }
    return __dadd_rn(first, rest);
}

template <int NV, bool MASS>
__device__ double slot_sum(const FemArgs &a, int p, int b, int *bad) {
    return reduceat_run(a.starts[p], a.starts[p + 1], [&](int q) -> double {
        const int o = a.order[q], e = o / (NV * NV), l = o - NV * NV * e;
        const Elem<NV> E = element<NV>(a.tri, a.V, a.vb, a.B, b, e);
        if (E.bad) atomicOr(bad, 1);
        const double c = (!MASS && a.coef) ? a.coef[(long long)e * a.cb + (a.cb > 1 ? b : 0)] : 1.0;
        return entry<MASS>(E, l / NV, l % NV, c, !MASS && a.coef);
    });
}

template <int NV>
__global__ void __launch_bounds__(256) fem_assemble_kernel(FemArgs a, int *bad) {
    const long long total = (long long)a.nnz * a.B;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int p = (int)(t / a.B), b = (int)(t - (long long)p * a.B);
        double v;
        if (a.mode == FEM_K) {
            v = slot_sum<NV, false>(a, p, b, bad);
        } else if (a.mode == FEM_M) {
            v = slot_sum<NV, true>(a, p, b, bad);
        } else {  // M + s K  (heat: dt * alpha, wave: dt * dt)
            v = __dadd_rn(slot_sum<NV, true>(a, p, b, bad), __dmul_rn(a.scale, slot_sum<NV, false>(a, p, b, bad)));
        }
        a.out[t] = v;
    }
}

// Shared vertices (one mesh for the batch), two passes:
//  prep  -- one thread per triplet: its unscaled stiffness and mass entries
//           (geometry and divides once per mesh, not per system) into kq / mq,
//           then one thread per slot sums the mass run into ms[p];
//  batch -- one thread per (slot, system), system fastest: the coefficient
//           products of the run summed in numpy's order. A warp's kq / order
//           reads are broadcasts, its coefficient reads and value stores are
//           contiguous.
template <int NV>
__global__ void __launch_bounds__(256) fem_prep_kernel(FemArgs a, int *bad) {
    const int m = NV * NV * a.nt;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < m; q += gridDim.x * blockDim.x) {
        const int o = a.order[q], e = o / (NV * NV), l = o - NV * NV * e;
        const Elem<NV> E = element<NV>(a.tri, a.V, 1, a.B, 0, e);
        if (E.bad) atomicOr(bad, 1);
        a.kq[q] = entry<false>(E, l / NV, l % NV, 1.0, false);
        if (a.mode != FEM_K) a.mq[q] = entry<true>(E, l / NV, l % NV, 1.0, false);
    }
}

// mass sum per slot from the per-triplet entries, numpy reduceat order
__global__ void __launch_bounds__(256) fem_mass_kernel(FemArgs a) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < a.nnz; p += gridDim.x * blockDim.x)
        a.ms[p] = reduceat_run(a.starts[p], a.starts[p + 1], [&](int q) -> double { return a.mq[q]; });
}

// value of item t = (slot p, system b) by the generic run walk (runs > 8)
__device__ double batch_item_slow(const FemArgs &a, unsigned p, unsigned b) {
    if (a.mode == FEM_M) return a.ms[p];
    const double Ks = reduceat_run(a.starts[p], a.starts[p + 1], [&](int q) -> double {
        const double k = a.kq[q];
        if (!a.coef) return k;
        return __dmul_rn(k, __ldg(&a.coef[(long long)(a.order[q] / a.nper2) * a.cb + (a.cb > 1 ? b : 0)]));
    });
    return a.mode == FEM_K ? Ks : __dadd_rn(a.ms[p], __dmul_rn(a.scale, Ks));
}

// A warp per slot, lanes over the systems: the run's stiffness entries and
// element ids are warp-uniform loads, each coefficient row a contiguous
// 256-byte load across the lanes, the values one contiguous store. Runs
// longer than 8 take the generic walk.
__global__ void __launch_bounds__(256, 8) fem_batch_kernel(FemArgs a) {  // 32 registers: full occupancy, the loads are latency-bound
    const int lane = threadIdx.x & 31;
    const int warps = gridDim.x * (blockDim.x >> 5);
    for (int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); p < a.nnz; p += warps) {
        const int q0 = a.starts[p], n = a.starts[p + 1] - q0;
        double *o = a.out + (long long)p * a.B;
        if (a.mode == FEM_M || n > 8) {
            for (int b = lane; b < a.B; b += 32) o[b] = batch_item_slow(a, (unsigned)p, (unsigned)b);
            continue;
        }
        const double msv = a.mode != FEM_K ? a.ms[p] : 0.0;
        for (int b0 = 0; b0 < a.B; b0 += 32) {
            const int b = b0 + lane;
            const int bc = a.cb > 1 ? min(b, a.B - 1) : 0;
            // run entries and element ids are warp-uniform loads; the coefficient
            // row is one contiguous load across the lanes
            auto term = [&](int q) -> double {
                const double k = __ldg(&a.kq[q]);
                return a.coef ? __dmul_rn(k, __ldg(&a.coef[(long long)(__ldg(&a.order[q]) / a.nper2) * a.cb + bc])) : k;
            };
            const double first = term(q0);
            double rest = -0.0;  // numpy's short sum (below 8 terms): sequential from -0.0
#pragma unroll 2
            for (int q = q0 + 1; q < q0 + n; ++q) rest = __dadd_rn(rest, term(q));
            const double Ks = __dadd_rn(first, rest);
            if (b < a.B) o[b] = a.mode == FEM_K ? Ks : __dadd_rn(msv, __dmul_rn(a.scale, Ks));
        }
    }
}

}  // namespace

std::string fem_plan_build(long long nv, long long nt, int nper, const long long *tri, FemPlanHost &h) {
    if (nv < 1 || nt < 1) return "empty mesh";
    if (nper != 3 && nper != 4) return "elements must be triangles (3 vertices) or tetrahedra (4)";
    const int n2 = nper * nper;
    if (nt * n2 > (long long)INT32_MAX || nv > (long long)INT32_MAX / 3) return "mesh too large for int32 plan";
    for (long long q = 0; q < nper * nt; ++q)
        if (tri[q] < 0 || tri[q] >= nv) return "element vertex out of range";
    const long long m = n2 * nt;
    std::vector<int> ord(m);
    std::iota(ord.begin(), ord.end(), 0);
    auto row = [&](int o) { return tri[nper * (long long)(o / n2) + (o % n2) / nper]; };
    auto col = [&](int o) { return tri[nper * (long long)(o / n2) + (o % n2) % nper]; };
    // np.lexsort((cols, rows)): by row, then column, ties in triplet order (stable)
    std::stable_sort(ord.begin(), ord.end(), [&](int u, int v) {
        const long long ru = row(u), rv = row(v);
        return ru != rv ? ru < rv : col(u) < col(v);
    });
    h.order = ord;
    h.starts.clear();
    h.col.clear();
    h.row_ptr.assign(nv + 1, 0);
    for (long long q = 0; q < m; ++q) {
        const int o = ord[q];
        if (q == 0 || row(o) != row(ord[q - 1]) || col(o) != col(ord[q - 1])) {
            h.starts.push_back((int)q);
            h.col.push_back(col(o));
            h.row_ptr[row(o) + 1] += 1;
        }
    }
    h.starts.push_back((int)m);
    for (long long i = 0; i < nv; ++i) h.row_ptr[i + 1] += h.row_ptr[i];
    for (size_t k = 0; k + 1 < h.starts.size(); ++k)
        if (h.starts[k + 1] - h.starts[k] > 129) return "more than 129 contributions to one entry";
    return "";
}

cudaError_t launch_fem_assemble(const FemArgs &a, int *bad, cudaStream_t s) {
    const long long total = (long long)a.nnz * a.B;
    if (total == 0) return cudaSuccess;
    note_launch();
    if (a.nper2 != 9 && a.nper2 != 16) return cudaErrorInvalidValue;
    if (a.vb == 1 && total < (1LL << 31)) {  // one mesh: per-slot geometry shared by the batch
        const int pg = (int)std::min<long long>(((long long)a.nper2 * a.nt + 255) / 256, 32LL * num_sms());
        if (a.nper2 == 9) fem_prep_kernel<3><<<pg, 256, 0, s>>>(a, bad);
        else fem_prep_kernel<4><<<pg, 256, 0, s>>>(a, bad);
        if (a.mode != FEM_K) {
            note_launch();
            fem_mass_kernel<<<(int)std::min<long long>((a.nnz + 255) / 256, 16LL * num_sms()), 256, 0, s>>>(a);
        }
        note_launch();
        fem_batch_kernel<<<(int)std::min<long long>((a.nnz + 7) / 8, 32LL * num_sms()), 256, 0, s>>>(a);
        return cudaGetLastError();
    }
    const int grid = (int)std::min<long long>((total + 255) / 256, 16LL * num_sms());
    if (a.nper2 == 9) fem_assemble_kernel<3><<<grid, 256, 0, s>>>(a, bad);
    else fem_assemble_kernel<4><<<grid, 256, 0, s>>>(a, bad);
    return cudaGetLastError();
}

}  // namespace npcg
