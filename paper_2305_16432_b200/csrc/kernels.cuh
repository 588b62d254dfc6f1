// kernels.cuh -- launch-side declarations of the PCG-path kernels (internal).
#pragma once
#include <algorithm>

#include "common.cuh"
#include "pattern.h"
#include "trsv.cuh"

namespace npcg {

constexpr int kSpmvThreads = 256;
constexpr int kMaxBatch = 256;   // columns per solver call
constexpr int kMaxCpl = 8;       // columns per lane (kMaxBatch / 32)
constexpr int kReduceBlocksPerSm = 2;

enum SpmvOp : int {
    SPMV_PLAIN = 0,        // Y = A X
    SPMV_APDOT = 1,        // Y = A P, partial p.Ap, alpha epilogue
    SPMV_RESID_INIT = 2,   // R = B - A X (or B), ||r||, initial record
    SPMV_RESID_DRIFT = 3,  // R = B - A X for drifted columns, convergence decision
    SPMV_RESID_FINAL = 4,  // ||B - A X|| for max-iter columns
};

struct SpmvArgs {
    int n = 0, B = 1;
    const int *rp = nullptr, *col = nullptr;
    const double *vals = nullptr;
    int vb = 0;  // values batched [nnz*B]
    const double *X = nullptr;
    double *Y = nullptr;
    const double *Bv = nullptr;
    double *R = nullptr;
    const double *P = nullptr;  // drift check: x + alpha p for columns with a pending update
    int op = SPMV_PLAIN;
    int has_x = 1;
    SolveState st{};
    double *partial = nullptr;
    Ctl *ctl = nullptr;
    int *drift_count = nullptr;
    int nslot = 0;
    // line-order ELL (ecol != null): every operand [b][nslot], see spmv_ell_kernel
    const int *ecol = nullptr;
    const double *evals = nullptr;
    // APDOT only: columns in PH_DRIFT compute their true residual R = Bv - A X2
    // in the same launch (the drift check of the previous pass, pcg.py:147-165)
    int merge_drift = 0;
    const double *X2 = nullptr;
    int ell_width = 0;
    size_t partial_cap = 0;  // doubles available at `partial`
};

__global__ void init_state_kernel(SolveState st, int B, long long hist_cap_init);
__global__ void normb_kernel(int n, int B, const double *v, SolveState st, double *partial, Ctl *ctl);
__global__ void init_x_kernel(long long nB, int B, const double *x0, double *x, SolveState st);
__global__ void pupd_kernel(long long nB, int B, double *z, double *p, double *x, SolveState st, int rearm);
__global__ void count_active_kernel(SolveState st, int B, long long *kmax, int finish);
__global__ void factor_from_lower_kernel(int nnz_lower, int B, int lb, const int *lower_slot,
                                         const int *pair, const double *lower, double *S);
__global__ void factor_to_lower_kernel(int nnz_lower, int B, const int *lower_slot, const double *S,
                                       double *lower);
__global__ void symmetric_check_kernel(long long nnz, int B, int vb, const int *pair, const double *vals,
                                       int *ok);

cudaError_t launch_spmv(const SpmvArgs &a, cudaStream_t s);
// line-order helpers (vectors [b][slot], see pattern.h LineSched)
cudaError_t launch_to_line(int nslot, int B, const int *rowof, const double *src, int src_batched, double pad,
                           double *dst, cudaStream_t s);
cudaError_t launch_from_line(int nslot, int B, const int *rowof, const double *src, double *dst, cudaStream_t s);
// all-line-order PCG vectors: p / x update, and value gathers into a packed order
cudaError_t launch_xupd_ell(int nslot, int B, const double *p, double *x, const SolveState &st, cudaStream_t s);
cudaError_t launch_pupd_ell(int nslot, int B, const double *z, double *p, double *x, const SolveState &st,
                            cudaStream_t s);
void launch_gather_rows(long long count, int B, const int *sel, const double *src, double *dst, cudaStream_t s);
void launch_gather_pack(long long per, int B, int sb, long long ps, long long bs, const int *perm, const double *S,
                        double *packed, cudaStream_t s);

}  // namespace npcg
