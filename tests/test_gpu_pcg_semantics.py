"""Solver semantics on the device loop, case for case with the reference's
own solver tests (pkg/tests/test_pcg.py:22-177, test_sparse.py:68-162,
test_gnn.py:113-228). Matrices are built by local helpers."""
import numpy as np
import pytest

from oracle import port
from paper_2305_16432_b200 import gnn, pcg, preconditioners, sparse
from paper_2305_16432_b200.errors import BreakdownError, DimensionMismatchError, NotSpdError
from paper_2305_16432_b200.sparse import LowerFactor, SparseMatrixCsr

pytestmark = pytest.mark.gpu


def spd_dense(n, rng, shift=None):
    m = rng.standard_normal((n, n))
    a = m @ m.T
    return (a + a.T) / 2.0 + (n if shift is None else shift) * np.eye(n)


def spd_sparse(n, rng, density=0.3):
    mask = np.triu(rng.random((n, n)) < density, 1)
    vals = rng.uniform(-1.0, 1.0, size=(n, n)) * mask
    sym = vals + vals.T
    return SparseMatrixCsr.from_dense(sym + np.diag(np.abs(sym).sum(axis=1) + rng.uniform(0.5, 1.5, size=n)))


def grid_laplacian(k):
    rows, cols, vals = [], [], []
    for i in range(k):
        for j in range(k):
            me = i * k + j
            for di, dj, v in ((0, 0, 4.0), (-1, 0, -1.0), (1, 0, -1.0), (0, -1, -1.0), (0, 1, -1.0)):
                ii, jj = i + di, j + dj
                if 0 <= ii < k and 0 <= jj < k:
                    rows.append(me)
                    cols.append(ii * k + jj)
                    vals.append(v)
    return SparseMatrixCsr.from_coo(k * k, rows, cols, vals)


def exact_factor(Ad):
    """Dense LDL^T (unit lower) as a LowerFactor."""
    n = Ad.shape[0]
    L = np.eye(n)
    d = np.zeros(n)
    W = Ad.copy()
    for j in range(n):
        d[j] = W[j, j]
        L[j + 1:, j] = W[j + 1:, j] / d[j]
        W[j + 1:, j + 1:] -= np.outer(L[j + 1:, j], W[j, j + 1:])
    r, c = np.tril_indices(n, -1)
    return LowerFactor(n, SparseMatrixCsr.from_coo(n, r, c, L[r, c]), d)


def test_identity_matrix_converges_immediately(gpu):
    A = SparseMatrixCsr.identity(7)
    b = np.arange(1.0, 8.0)
    x, rep = pcg.pcg_solve(A, b)
    assert rep.converged and rep.iterations <= 1
    np.testing.assert_allclose(x, b, rtol=0, atol=1e-15)


def test_two_by_two(gpu):
    A = SparseMatrixCsr.from_dense(np.array([[2.0, 0.0], [0.0, 2.0]]))
    x, rep = pcg.pcg_solve(A, np.array([2.0, 4.0]))
    assert rep.iterations <= 2 and rep.converged
    np.testing.assert_allclose(x, [1.0, 2.0], atol=1e-14)


def test_exact_factor_converges_in_two(gpu):
    rng = np.random.default_rng(3)
    Ad = spd_dense(50, rng)
    A = SparseMatrixCsr.from_dense(Ad)
    b = rng.standard_normal(50)
    P = preconditioners.FactorPreconditioner("ic0", exact_factor(Ad))
    x, rep = pcg.pcg_solve(A, b, P)
    assert rep.converged and rep.iterations <= 2
    assert np.linalg.norm(b - Ad @ x) <= 1e-12 * np.linalg.norm(b)


def test_matches_dense_solve(gpu):
    rng = np.random.default_rng(11)
    Ad = spd_dense(40, rng)
    b = rng.standard_normal(40)
    x, rep = pcg.pcg_solve(SparseMatrixCsr.from_dense(Ad), b)
    assert rep.converged
    assert np.max(np.abs(x - np.linalg.solve(Ad, b))) < 1e-8


@pytest.mark.parametrize("n,seed", [(2, 0), (5, 1), (17, 2), (30, 3)])
def test_finite_termination(gpu, n, seed):
    rng = np.random.default_rng(seed)
    Ad = spd_dense(n, rng)
    b = rng.standard_normal(n)
    _, rep = pcg.pcg_solve(SparseMatrixCsr.from_dense(Ad), b, opts=pcg.SolveOptions(thresholds=(1e-10,)))
    assert rep.converged and rep.iterations <= n + 5


def test_foreign_preconditioner_sees_positive_energy(gpu):
    rng = np.random.default_rng(5)
    A = grid_laplacian(6)
    b = rng.standard_normal(A.n)
    seen = []

    class Recorder:
        def apply_inverse(self, r):
            z = r / 4.0
            seen.append(float(r @ z))
            return z

    _, rep = pcg.pcg_solve(A, b, Recorder())
    assert rep.converged
    assert all(v > 0.0 for v in seen[:-1])


def test_zero_rhs(gpu):
    A = grid_laplacian(4)
    x, rep = pcg.pcg_solve(A, np.zeros(A.n), opts=pcg.SolveOptions(x0=np.ones(A.n)))
    assert rep.converged and rep.iterations == 0
    assert np.all(x == 0.0)
    assert rep.iterations_to[1e-12] == 0
    assert rep.history == [0.0]


def test_thresholds_monotone_and_history_length(gpu):
    rng = np.random.default_rng(9)
    A = grid_laplacian(10)
    b = rng.standard_normal(A.n)
    _, rep = pcg.pcg_solve(A, b)
    iters = [rep.iterations_to[t] for t in rep.thresholds]
    assert iters == sorted(iters)
    assert all(rep.seconds_to[t] >= 0.0 for t in rep.thresholds)
    assert len(rep.history) == rep.iterations + 1


def test_max_iter_exhaustion(gpu):
    rng = np.random.default_rng(2)
    A = grid_laplacian(12)
    b = rng.standard_normal(A.n)
    x, rep = pcg.pcg_solve(A, b, opts=pcg.SolveOptions(max_iter=3))
    assert not rep.converged and rep.iterations == 3
    assert np.linalg.norm(b - A.to_dense() @ x) < np.linalg.norm(b)
    true_rel = np.linalg.norm(b - A.to_dense() @ x) / np.linalg.norm(b)
    assert rep.final_relative_residual == pytest.approx(true_rel, rel=1e-12)


def test_indefinite_breaks_down(gpu):
    A = SparseMatrixCsr.from_dense(np.array([[1.0, 0.0], [0.0, -1.0]]))
    with pytest.raises(BreakdownError):
        pcg.pcg_solve(A, np.array([1.0, 1.0]))


def test_warm_start_exact(gpu):
    rng = np.random.default_rng(7)
    Ad = spd_dense(12, rng)
    xs = rng.standard_normal(12)
    b = Ad @ xs
    x, rep = pcg.pcg_solve(SparseMatrixCsr.from_dense(Ad), b, opts=pcg.SolveOptions(x0=xs))
    assert rep.iterations == 0 and rep.converged
    np.testing.assert_allclose(x, xs)


def test_absolute_mode(gpu):
    rng = np.random.default_rng(4)
    A = grid_laplacian(6)
    b = 1e-6 * rng.standard_normal(A.n)
    _, rel_rep = pcg.pcg_solve(A, b, opts=pcg.SolveOptions(thresholds=(1e-4,)))
    _, abs_rep = pcg.pcg_solve(A, b, opts=pcg.SolveOptions(thresholds=(1e-4,), absolute=True))
    assert abs_rep.iterations_to[1e-4] < rel_rep.iterations_to[1e-4]
    assert abs_rep.history[abs_rep.iterations_to[1e-4]] <= 1e-4


def test_final_residual_recomputed(gpu):
    rng = np.random.default_rng(13)
    A = grid_laplacian(9)
    b = rng.standard_normal(A.n)
    x, rep = pcg.pcg_solve(A, b)
    true_rel = np.linalg.norm(b - A.to_dense() @ x) / np.linalg.norm(b)
    assert true_rel <= 10 * max(rep.final_relative_residual, 1e-300)
    assert true_rel <= 1e-12


def test_options_validation():
    with pytest.raises(DimensionMismatchError):
        pcg.SolveOptions(thresholds=())
    with pytest.raises(DimensionMismatchError):
        pcg.SolveOptions(thresholds=(1e-4, 1e-2))
    with pytest.raises(DimensionMismatchError):
        pcg.SolveOptions(thresholds=(1.5,))
    with pytest.raises(DimensionMismatchError):
        pcg.SolveOptions(max_iter=0)


def test_rhs_shape_checked(gpu):
    with pytest.raises(DimensionMismatchError):
        pcg.pcg_solve(SparseMatrixCsr.identity(3), np.ones(4))


def test_jacobi_and_gauss_seidel_match_oracle(gpu):
    rng = np.random.default_rng(21)
    A = spd_sparse(60, rng, 0.1)
    b = rng.standard_normal(A.n)
    oA = port.Csr(A.n, A.row_ptr, A.col_idx, A.values)
    for kind in ("jacobi", "gauss_seidel", "identity"):
        P = preconditioners.build(kind, A)
        x, rep = pcg.pcg_solve(A, b, P)
        oF = port.Factor(A.n, port.Csr(A.n, P.factor.strict_lower.row_ptr, P.factor.strict_lower.col_idx,
                                       P.factor.strict_lower.values), P.factor.diag)
        ox, orep = port.pcg_solve(oA, b, oF)
        assert abs(rep.iterations - orep.iterations) <= 1
        assert np.linalg.norm(x - ox) <= 1e-8 * np.linalg.norm(ox)


def test_apply_inverse_roundtrip(gpu):
    for seed, n in ((0, 1), (1, 2), (2, 50), (3, 200)):
        rng = np.random.default_rng(seed)
        low = spd_sparse(n, rng).strict_lower() if n > 1 else SparseMatrixCsr.from_coo(1, [], [], [])
        if low.nnz:
            mass = np.abs(low.to_dense()).sum(axis=1)[low.row_indices()]
            low = SparseMatrixCsr(n, low.row_ptr, low.col_idx, low.values / (mass + 0.25))
        F = LowerFactor(n, low, rng.uniform(0.5, 3.0, size=n))
        x = rng.standard_normal(n)
        back = sparse.ldlt_apply_inverse(F, sparse.ldlt_apply(F, x))
        assert np.abs(back - x).max() <= 1e-10 * max(np.abs(x).max(), 1.0)


def test_apply_inverse_kats(gpu):
    empty = SparseMatrixCsr.from_coo(2, [], [], [])
    F = LowerFactor(2, empty, np.array([2.0, 4.0]))
    assert np.array_equal(sparse.ldlt_apply_inverse(F, np.array([2.0, 4.0])), [1.0, 1.0])
    F1 = LowerFactor(1, SparseMatrixCsr.from_coo(1, [], [], []), np.array([8.0]))
    assert sparse.ldlt_apply_inverse(F1, np.array([2.0]))[0] == 0.25


def test_spmv_kats(gpu):
    a = SparseMatrixCsr.identity(3)
    assert np.array_equal(sparse.spmv(a, np.array([1.0, 2.0, 3.0])), [1.0, 2.0, 3.0])
    e = SparseMatrixCsr.from_coo(4, [], [], [])
    assert np.array_equal(sparse.spmv(e, np.arange(4.0)), np.zeros(4))
    d = SparseMatrixCsr.from_dense([[2.0, 1.0], [1.0, 3.0]])
    assert np.array_equal(sparse.spmv(d, np.array([1.0, 1.0])), [3.0, 4.0])
    with pytest.raises(DimensionMismatchError):
        sparse.spmv(SparseMatrixCsr.identity(3), np.zeros(2))


SMALL = gnn.GnnHyperParams(l=1, h=8, n_mp=2, l_mp=1, h_mp=8)


def test_zero_decoder_is_jacobi(gpu):
    A = grid_laplacian(4)
    model = gnn.create_model(SMALL, seed=0)
    model.params[f"edge_dec.{SMALL.l}.w"][:] = 0.0
    P = gnn.build_learned(model, A, np.ones(A.n))
    np.testing.assert_array_equal(P.to_dense(), preconditioners.build_jacobi(A).to_dense())


def test_assemble_diagonal_system_exact(gpu):
    A = SparseMatrixCsr.from_dense(np.diag([4.0, 2.0, 9.0]))
    P = gnn.assemble_preconditioner(np.zeros(0), A)
    x, rep = pcg.pcg_solve(A, np.array([8.0, 2.0, 27.0]), P, pcg.SolveOptions(thresholds=(1e-12,)))
    assert rep.iterations <= 1
    np.testing.assert_allclose(x, [2.0, 1.0, 3.0], atol=1e-14)


def test_learned_solves_grid(gpu):
    A = grid_laplacian(7)
    b = np.random.default_rng(2).standard_normal(A.n)
    P = gnn.build_learned(gnn.create_model(SMALL, seed=4), A, b)
    x, rep = pcg.pcg_solve(A, b, P, pcg.SolveOptions(thresholds=(1e-10,)))
    assert rep.converged
    np.testing.assert_allclose(A.to_dense() @ x, b, atol=1e-8)


def test_not_spd_pivot(gpu):
    bad = SparseMatrixCsr.from_dense(np.array([[1.0, 0.5], [0.5, -2.0]]))
    with pytest.raises(NotSpdError) as err:
        gnn.build_learned(gnn.create_model(SMALL, seed=0), bad, np.ones(2))
    assert err.value.pivot == 1


def test_graph_rejects_bad_systems(gpu):
    from paper_2305_16432_b200.errors import DataFormatError
    hollow = SparseMatrixCsr.from_coo(2, [0, 1], [1, 0], [1.0, 1.0])
    with pytest.raises(DataFormatError):
        gnn.build_learned(gnn.create_model(SMALL, seed=0), hollow, np.zeros(2))
    skew = SparseMatrixCsr.from_dense(np.array([[1.0, 2.0], [0.5, 1.0]]))
    with pytest.raises(DataFormatError):
        gnn.build_learned(gnn.create_model(SMALL, seed=0), skew, np.zeros(2))


def test_deterministic_bitwise(gpu):
    A = spd_sparse(80, np.random.default_rng(0), 0.1)
    b = np.random.default_rng(1).standard_normal(80)
    model = gnn.create_model(gnn.GnnHyperParams(l=1, h=16, n_mp=3, l_mp=1, h_mp=16), seed=2)
    P1 = gnn.build_learned(model, A, b)
    P2 = gnn.build_learned(model, A, b)
    np.testing.assert_array_equal(P1.factor.strict_lower.values, P2.factor.strict_lower.values)
    x1, r1 = pcg.pcg_solve(A, b, P1)
    x2, r2 = pcg.pcg_solve(A, b, P2)
    np.testing.assert_array_equal(x1, x2)
    assert r1.history == r2.history


@pytest.mark.parametrize("k", [12, 40])
def test_non_finite_runs_to_max_iter(gpu, k):
    """SURVEY Appendix A.3 (pcg.py:136-140): an overflowing factor makes
    p'Ap inf / NaN; `pAp <= 0.0` is then False, so no BreakdownError -- the
    NaN propagates, the loop runs to max_iter and converged is False, with a
    NaN final residual. Checked against the oracle (the reference's own
    semantics); k = 40 takes the line-wavefront path, k = 12 the level path
    or the line path depending on the pattern."""
    from paper_2305_16432_b200 import inputs
    prob = inputs.heat_2d(k=k, cfg=13)
    A, b = prob.A, prob.rhs[:, 0]
    low = A.strict_lower()
    vals = np.where(np.arange(low.nnz) % 2 == 0, 1e300, -1e300)
    P = gnn.assemble_preconditioner(vals, A)
    oF = port.Factor(A.n, port.Csr(A.n, low.row_ptr, low.col_idx, vals), A.diagonal())
    with np.errstate(all="ignore"):
        ox, orep = port.pcg_solve(port.Csr(A.n, A.row_ptr, A.col_idx, A.values), b, oF,
                                  thresholds=(1e-8,), max_iter=25)
    x, rep = pcg.pcg_solve(A, b, P, pcg.SolveOptions(thresholds=(1e-8,), max_iter=25))
    assert orep.breakdown is None and not orep.converged and orep.iterations == 25
    assert not rep.converged and rep.iterations == 25
    assert rep.status == orep_status_maxiter()
    assert np.isnan(rep.final_relative_residual) == np.isnan(orep.final_relative_residual)
    assert len(rep.history) == 26


def orep_status_maxiter():
    from paper_2305_16432_b200 import _native
    return _native.STATUS_MAXITER


def test_reference_dataset_solves_on_device(gpu):
    """A dataset written by the reference (tests/golden/dataset_heat_small,
    fem.py:417-448): each pattern group solved as one batch on the device
    reproduces the stored x (the reference's own 1e-12 solves)."""
    import os
    from paper_2305_16432_b200 import datasets
    gold = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "dataset_heat_small")
    _, trajs = datasets.load_dataset(gold)
    tuples = [t for traj in trajs for t in traj.tuples]
    for group in datasets.group_by_pattern(tuples):
        A, values, rhs, x_ref = datasets.stack_tuples(group)
        P = preconditioners.build_jacobi(A) if values.shape[1] == 1 else None
        X, reps = pcg.pcg_solve_batch(A, rhs, P, pcg.SolveOptions(thresholds=(1e-12,)), values=values)
        for j, rep in enumerate(reps):
            assert rep.converged
            assert np.linalg.norm(X[:, j] - x_ref[:, j]) <= 1e-9 * np.linalg.norm(x_ref[:, j])
