/*
 * oracle/kernels.c -- CPU restatement of the reference's compiled kernels.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing on the product path links or calls this
 * file; it is the checker for tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py.
 *
 * The reference compiles these three loops with numba.njit
 * (pkg/src/pcgkit/sparse.py:213-239). They are restated here in plain C99
 * with the same summation order, int64 indices and float64 values, and
 * built with -ffp-contract=off so no fused multiply-add changes rounding:
 * the results are bitwise identical to the reference (pinned by
 * tests/test_oracle_golden.py against goldens produced by the reference).
 */
#include <stdint.h>

/* y = A x, rows ascending, entries in CSR order (sparse.py:213-219). */
void oracle_spmv(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                 const double *values, const double *x, double *y)
{
    for (int64_t i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p)
            acc += values[p] * x[col_idx[p]];
        y[i] = acc;
    }
}

/* (I + L) y = r, L strictly lower CSR, rows ascending (sparse.py:222-229). */
void oracle_forward_unit(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                         const double *values, const double *rhs, double *out)
{
    for (int64_t i = 0; i < n; ++i) {
        double acc = rhs[i];
        for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p)
            acc -= values[p] * out[col_idx[p]];
        out[i] = acc;
    }
}

/* (I + L)^T z = y in place, i descending, column scatter (sparse.py:232-239). */
void oracle_backward_unit_t(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                            const double *values, double *out)
{
    for (int64_t i = n - 1; i >= 0; --i) {
        const double zi = out[i];
        for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p)
            out[col_idx[p]] -= values[p] * zi;
    }
}

/* z = (I+L)^-T D^-1 (I+L)^-1 r (sparse.py:265-275), fused for speed. */
void oracle_ldlt_apply_inverse(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                               const double *values, const double *diag,
                               const double *r, double *z)
{
    oracle_forward_unit(n, row_ptr, col_idx, values, r, z);
    for (int64_t i = 0; i < n; ++i)
        z[i] /= diag[i];
    oracle_backward_unit_t(n, row_ptr, col_idx, values, z);
}
