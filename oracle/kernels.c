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
#include <stddef.h>
#include <stdlib.h>
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

/* Canonical-order segment sum (autodiff.py:221-243) for segments that are
 * contiguous runs of a non-decreasing `seg` (CSR-ordered edges, gnn.py:83):
 * inside a segment the addend rows are stably sorted lexicographically by
 * (x[:,0], x[:,1], ...) -- np.lexsort's order with seg as the primary key --
 * and summed as np.add.reduceat does along axis 0: the first row plus
 * numpy's pairwise sum of the rest (from -0.0 sequentially below 8 terms,
 * eight interleaved accumulators up to 128, halving above). Same arithmetic
 * as the numpy restatement, without the m-row lexsort over F+1 keys. Rows of
 * `out` with no addend are left untouched. */
static int lex_less(const double *a, const double *b, int64_t F)
{
    for (int64_t c = 0; c < F; ++c) {
        if (a[c] < b[c]) return 1;
        if (a[c] > b[c]) return 0;
        if (a[c] != a[c] && b[c] == b[c]) return 0; /* NaN sorts last */
        if (a[c] == a[c] && b[c] != b[c]) return 1;
    }
    return 0;
}

/* numpy pairwise_sum over rows r[0..n) of column c (rows are pointers) */
static double pairwise_col(const double *const *r, int64_t n, int64_t c)
{
    if (n < 8) {
        double res = -0.0;
        for (int64_t i = 0; i < n; ++i) res += r[i][c];
        return res;
    }
    if (n <= 128) {
        double a[8];
        for (int j = 0; j < 8; ++j) a[j] = r[j][c];
        int64_t i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) a[j] += r[i + j][c];
        double res = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
        for (; i < n; ++i) res += r[i][c];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise_col(r, n2, c) + pairwise_col(r + n2, n - n2, c);
}

void oracle_segment_sum_sorted(int64_t m, int64_t F, const double *x, const int64_t *seg, double *out)
{
    int64_t s = 0;
    int64_t cap = 64;
    int64_t *idx = (int64_t *)malloc((size_t)cap * sizeof(int64_t));
    const double **rows = (const double **)malloc((size_t)cap * sizeof(double *));
    while (s < m) {
        int64_t e = s + 1;
        while (e < m && seg[e] == seg[s]) ++e;
        const int64_t cnt = e - s;
        if (cnt > cap) {
            cap = cnt;
            idx = (int64_t *)realloc(idx, (size_t)cap * sizeof(int64_t));
            rows = (const double **)realloc(rows, (size_t)cap * sizeof(double *));
        }
        /* stable insertion sort of the segment's rows */
        for (int64_t k = 0; k < cnt; ++k) {
            int64_t j = k;
            while (j > 0 && lex_less(x + (s + k) * F, x + idx[j - 1] * F, F)) {
                idx[j] = idx[j - 1];
                --j;
            }
            idx[j] = s + k;
        }
        for (int64_t k = 0; k < cnt; ++k) rows[k] = x + idx[k] * F;
        double *o = out + seg[s] * F;
        for (int64_t c = 0; c < F; ++c) o[c] = cnt > 1 ? rows[0][c] + pairwise_col(rows + 1, cnt - 1, c) : rows[0][c];
        s = e;
    }
    free(idx);
    free(rows);
}
