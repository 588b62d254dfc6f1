"""Configs 4 and 5 (3-D Kuhn cubes, P1 tetrahedra) at parity-test sizes:
the triangular solves take the level-set path (3-D patterns have no line
schedule), the GNN runs on ~12 neighbours per row. Checker: the oracle port
(pinned to pcgkit on the goldens). Bars as in test_gpu_parity.py."""
import numpy as np
import pytest

from oracle import port
from paper_2305_16432_b200 import gnn, inputs, pcg, sparse

pytestmark = pytest.mark.gpu

L_TOL = 1e-5
X_TOL = 1e-8


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def perturbed_model(seed, h=16, n_mp=2):
    hyper = gnn.GnnHyperParams(l=1, h=h, n_mp=n_mp, l_mp=1, h_mp=h)
    model = gnn.create_model(hyper, seed=seed)
    for r in range(hyper.n_mp):  # cancel the processor output gain: non-trivial L'
        for s in ("node", "edge"):
            model.params[f"mp{r}.{s}.1.w"] *= 10.0
    return model, port.Hyper(l=1, h=h, n_mp=n_mp, l_mp=1, h_mp=h)


def test_apply_inverse_bitwise_3d(gpu):
    A = inputs.poisson_3d(k=10, batch=1).A
    rng = np.random.default_rng(7)
    low = A.strict_lower()
    vals = rng.uniform(-0.2, 0.2, size=low.nnz)
    F = sparse.LowerFactor(A.n, sparse.SparseMatrixCsr(A.n, low.row_ptr, low.col_idx, vals), A.diagonal())
    oF = port.Factor(A.n, port.Csr(A.n, low.row_ptr, low.col_idx, vals), A.diagonal())
    for s in range(3):
        r = rng.standard_normal(A.n)
        np.testing.assert_array_equal(sparse.ldlt_apply_inverse(F, r), oF.apply_inverse(r))
    x = rng.standard_normal(A.n)
    np.testing.assert_array_equal(sparse.spmv(A, x), port.spmv(port.Csr(A.n, A.row_ptr, A.col_idx, A.values), x))


def test_poisson_3d_shared_factor_batch(gpu):
    """Config-4 shape: one L' from the GNN on RHS 0, a batch of GRF loads."""
    prob = inputs.poisson_3d(k=9, batch=6)
    A = prob.A
    oA = port.Csr(A.n, A.row_ptr, A.col_idx, A.values)
    model, ohp = perturbed_model(0)
    P = gnn.build_learned(model, A, prob.rhs[:, 0])
    oF = port.build_learned(ohp, model.params, oA, prob.rhs[:, 0])
    assert rel(P.factor.strict_lower.values, oF.lower.values) <= L_TOL
    thr = (1e-8,)
    X, reps = pcg.pcg_solve_batch(A, prob.rhs, P, pcg.SolveOptions(thresholds=thr, max_iter=3000))
    for s, rep in enumerate(reps):
        ox, orep = port.pcg_solve(oA, prob.rhs[:, s], oF, thresholds=thr, max_iter=3000)
        assert rep.converged and orep.converged
        assert abs(rep.iterations - orep.iterations) <= 1, (s, rep.iterations, orep.iterations)
        assert rel(X[:, s], ox) <= X_TOL


def test_heat_3d_distinct_systems(gpu):
    """Config-5 shape: distinct A (per-element exp(GRF) diffusivity) and L' per
    system, rtol 1e-10."""
    prob = inputs.heat_3d(k=7, batch=3)
    A, vals = prob.A, prob.values
    model, ohp = perturbed_model(1)
    P = gnn.build_learned_batch(model, A, prob.rhs, values=vals)
    thr = (1e-10,)
    X, reps = pcg.pcg_solve_batch(A, prob.rhs, P, pcg.SolveOptions(thresholds=thr, max_iter=3000), values=vals)
    for s, rep in enumerate(reps):
        oA = port.Csr(A.n, A.row_ptr, A.col_idx, np.ascontiguousarray(vals[:, s]))
        oF = port.build_learned(ohp, model.params, oA, prob.rhs[:, s])
        assert rel(P.system_factor(s).strict_lower.values, oF.lower.values) <= L_TOL
        ox, orep = port.pcg_solve(oA, prob.rhs[:, s], oF, thresholds=thr, max_iter=3000)
        assert rep.converged and orep.converged
        assert abs(rep.iterations - orep.iterations) <= 1, (s, rep.iterations, orep.iterations)
        assert rel(X[:, s], ox) <= X_TOL


# ---- level-synchronous solves (trsv_level.cu): forced on at test sizes ----


@pytest.fixture
def levelsync(monkeypatch):
    monkeypatch.setenv("NPCG_LEVELSYNC", "1")


def test_poisson_3d_trained_checkpoint(gpu, levelsync, monkeypatch):
    """tools/bench_3d.py's config-4 weights (weights/poisson3d_latent64_mp5.json,
    trained by the device training step on 6^3 .. 12^3 cubes): latent-64
    tensor-core GNN + level-path PCG against the oracle on a 14^3 cube, and the
    trained factor beats Jacobi by a wide margin."""
    import os

    import torch

    from paper_2305_16432_b200 import preconditioners
    monkeypatch.setattr(gnn, "FEATURE_WIDTH", 64)
    path = os.path.join(os.path.dirname(os.path.abspath(gnn.__file__)), "weights", "poisson3d_latent64_mp5.json")
    model = gnn.load_model(path)
    ohp = port.Hyper(l=1, h=model.hyper.h, n_mp=model.hyper.n_mp, l_mp=1, h_mp=model.hyper.h_mp, width=64)
    prob = inputs.poisson_3d(k=14, batch=6)
    A = prob.A
    P = gnn.build_learned(model, A, prob.rhs[:, 0])
    oA = port.Csr(A.n, A.row_ptr, A.col_idx, A.values)
    oF = port.build_learned(ohp, model.params, oA, prob.rhs[:, 0])
    assert rel(P.factor.strict_lower.values, oF.lower.values) <= L_TOL
    thr = (1e-8,)
    X, reps = pcg.pcg_solve_batch(A, torch.from_numpy(prob.rhs).cuda(), P, pcg.SolveOptions(thresholds=thr, max_iter=2000))
    X = X.cpu().numpy()
    _, jac = pcg.pcg_solve(A, prob.rhs[:, 0], preconditioners.build_jacobi(A), pcg.SolveOptions(thresholds=thr))
    for s in (0, 3, 5):
        ox, orep = port.pcg_solve(oA, prob.rhs[:, s], oF, thresholds=thr, max_iter=2000)
        assert reps[s].converged and orep.converged
        assert abs(reps[s].iterations - orep.iterations) <= 1, (s, reps[s].iterations, orep.iterations)
        assert rel(X[:, s], ox) <= X_TOL
    assert 3 * max(r.iterations for r in reps) < jac.iterations


def test_heat_3d_trained_checkpoint(gpu, levelsync, monkeypatch):
    """Config 5's weights (weights/heat3d_latent64_mp5.json: trained on small
    cubes with dt scaled to config 5's mass : stiffness balance): distinct
    systems, per-system L' from the tensor-core GNN, rtol 1e-10, against the
    oracle."""
    import os
    monkeypatch.setattr(gnn, "FEATURE_WIDTH", 64)
    path = os.path.join(os.path.dirname(os.path.abspath(gnn.__file__)), "weights", "heat3d_latent64_mp5.json")
    model = gnn.load_model(path)
    ohp = port.Hyper(l=1, h=model.hyper.h, n_mp=model.hyper.n_mp, l_mp=1, h_mp=model.hyper.h_mp, width=64)
    prob = inputs.heat_3d(k=12, batch=3, dt=1e-3 * (128.0 / 12) ** 2)
    A, vals = prob.A, prob.values
    P = gnn.build_learned_batch(model, A, prob.rhs, values=vals)
    thr = (1e-10,)
    X, reps = pcg.pcg_solve_batch(A, prob.rhs, P, pcg.SolveOptions(thresholds=thr, max_iter=3000), values=vals)
    for s, rep in enumerate(reps):
        oA = port.Csr(A.n, A.row_ptr, A.col_idx, np.ascontiguousarray(vals[:, s]))
        oF = port.build_learned(ohp, model.params, oA, prob.rhs[:, s])
        assert rel(P.system_factor(s).strict_lower.values, oF.lower.values) <= L_TOL
        ox, orep = port.pcg_solve(oA, prob.rhs[:, s], oF, thresholds=thr, max_iter=3000)
        assert rep.converged and orep.converged
        assert abs(rep.iterations - orep.iterations) <= 1, (s, rep.iterations, orep.iterations)
        assert rel(X[:, s], ox) <= X_TOL


def test_level_sync_apply_inverse_bitwise(gpu, levelsync):
    import torch
    A = inputs.poisson_3d(k=9, batch=1).A
    rng = np.random.default_rng(11)
    low = A.strict_lower()
    vals = rng.uniform(-0.2, 0.2, size=low.nnz)
    F = sparse.LowerFactor(A.n, sparse.SparseMatrixCsr(A.n, low.row_ptr, low.col_idx, vals), A.diagonal())
    oF = port.Factor(A.n, port.Csr(A.n, low.row_ptr, low.col_idx, vals), A.diagonal())
    r = rng.standard_normal(A.n)
    np.testing.assert_array_equal(sparse.ldlt_apply_inverse(F, r), oF.apply_inverse(r))
    # a batch of 40 right-hand sides through the device entry point
    R = rng.standard_normal((A.n, 40))
    P = gnn.assemble_preconditioner(vals, A)
    Z = P.apply_inverse(torch.from_numpy(R).cuda()).cpu().numpy()
    for j in (0, 17, 39):
        np.testing.assert_array_equal(Z[:, j], oF.apply_inverse(R[:, j]))


def test_level_sync_shared_factor_batch(gpu, levelsync):
    """Config-4 shape through the level-synchronous kernels."""
    prob = inputs.poisson_3d(k=9, batch=24)
    A = prob.A
    oA = port.Csr(A.n, A.row_ptr, A.col_idx, A.values)
    model, ohp = perturbed_model(0)
    P = gnn.build_learned(model, A, prob.rhs[:, 0])
    oF = port.build_learned(ohp, model.params, oA, prob.rhs[:, 0])
    thr = (1e-8,)
    X, reps = pcg.pcg_solve_batch(A, prob.rhs, P, pcg.SolveOptions(thresholds=thr, max_iter=3000))
    for s in (0, 7, 23):
        ox, orep = port.pcg_solve(oA, prob.rhs[:, s], oF, thresholds=thr, max_iter=3000)
        assert reps[s].converged and orep.converged
        assert abs(reps[s].iterations - orep.iterations) <= 1, (s, reps[s].iterations, orep.iterations)
        assert rel(X[:, s], ox) <= X_TOL
    # decoupled from the GNN: the oracle's own L', the first residual norms agree
    # up to the dot products' summation order
    Po = gnn.assemble_preconditioner(oF.lower.values, A)
    X2, reps2 = pcg.pcg_solve_batch(A, prob.rhs, Po, pcg.SolveOptions(thresholds=thr, max_iter=3000))
    ox, orep = port.pcg_solve(oA, prob.rhs[:, 5], oF, thresholds=thr, max_iter=3000)
    np.testing.assert_allclose(np.array(reps2[5].history)[:4], np.array(orep.history)[:4], rtol=1e-9)
    assert abs(reps2[5].iterations - orep.iterations) <= 1


def test_level_sync_distinct_systems(gpu, levelsync):
    """Config-5 shape (per-system A and L', rtol 1e-10) through the
    level-synchronous kernels."""
    prob = inputs.heat_3d(k=7, batch=5)
    A, vals = prob.A, prob.values
    model, ohp = perturbed_model(1)
    P = gnn.build_learned_batch(model, A, prob.rhs, values=vals)
    thr = (1e-10,)
    X, reps = pcg.pcg_solve_batch(A, prob.rhs, P, pcg.SolveOptions(thresholds=thr, max_iter=3000), values=vals)
    for s, rep in enumerate(reps):
        oA = port.Csr(A.n, A.row_ptr, A.col_idx, np.ascontiguousarray(vals[:, s]))
        oF = port.build_learned(ohp, model.params, oA, prob.rhs[:, s])
        ox, orep = port.pcg_solve(oA, prob.rhs[:, s], oF, thresholds=thr, max_iter=3000)
        assert rep.converged and orep.converged
        assert abs(rep.iterations - orep.iterations) <= 1, (s, rep.iterations, orep.iterations)
        assert rel(X[:, s], ox) <= X_TOL


# ---- the walk variants (trsv_level.cu): dependency flags (warp per row for
# B a multiple of 32 dividing into <= 8 warps, thread per column otherwise)
# and the barrier-per-level walk; every one bitwise the oracle's solves ----


@pytest.mark.parametrize("flags", ["1", "0"])
@pytest.mark.parametrize("B", [1, 5, 32, 64, 96, 128, 256])
def test_level_walk_apply_inverse_bitwise(gpu, levelsync, monkeypatch, B, flags):
    import torch
    monkeypatch.setenv("NPCG_LEVELFLAGS", flags)
    A = inputs.poisson_3d(k=7, batch=1).A
    rng = np.random.default_rng(100 + B)
    low = A.strict_lower()
    vals = rng.uniform(-0.2, 0.2, size=low.nnz)
    oF = port.Factor(A.n, port.Csr(A.n, low.row_ptr, low.col_idx, vals), A.diagonal())
    R = rng.standard_normal((A.n, B))
    P = gnn.assemble_preconditioner(vals, A)
    Z = P.apply_inverse(torch.from_numpy(R).cuda()).cpu().numpy()
    for j in sorted({0, B // 2, B - 1}):
        np.testing.assert_array_equal(Z[:, j], oF.apply_inverse(R[:, j]))


@pytest.mark.parametrize("B", [32, 128])
def test_level_walk_pcg_flags_vs_barrier(gpu, levelsync, monkeypatch, B):
    """Shared factor, B columns: the flag walk and the barrier walk solve the
    same systems (their dot products sum in different fixed orders)."""
    prob = inputs.poisson_3d(k=8, batch=B)
    A = prob.A
    rng = np.random.default_rng(B)
    vals = rng.uniform(-0.15, 0.0, size=A.strict_lower().nnz)
    thr = (1e-8,)
    out = {}
    for flags in ("1", "0"):
        monkeypatch.setenv("NPCG_LEVELFLAGS", flags)
        P = gnn.assemble_preconditioner(vals, A)
        out[flags] = pcg.pcg_solve_batch(A, prob.rhs, P, pcg.SolveOptions(thresholds=thr, max_iter=3000))
    (X1, r1), (X0, r0) = out["1"], out["0"]
    for s in range(B):
        assert r1[s].converged and r0[s].converged
        assert abs(r1[s].iterations - r0[s].iterations) <= 1, (s, r1[s].iterations, r0[s].iterations)
        assert rel(X1[:, s], X0[:, s]) <= X_TOL
    oA = port.Csr(A.n, A.row_ptr, A.col_idx, A.values)
    low = A.strict_lower()
    oF = port.Factor(A.n, port.Csr(A.n, low.row_ptr, low.col_idx, vals), A.diagonal())
    ox, orep = port.pcg_solve(oA, prob.rhs[:, B - 1], oF, thresholds=thr, max_iter=3000)
    assert abs(r1[B - 1].iterations - orep.iterations) <= 1
    assert rel(X1[:, B - 1], ox) <= X_TOL


def test_level_walk_distinct_systems_warp_rows(gpu, levelsync, monkeypatch):
    """Per-system A and L' at B = 64 (warp per row, two columns per lane,
    factor values [entry][B]): the flag walk against the barrier walk on every
    column, and against the oracle on systems 0-4 (the conditioning the batch-5
    test above pins)."""
    prob = inputs.heat_3d(k=7, batch=64)
    A, vals = prob.A, prob.values
    model, ohp = perturbed_model(1)
    thr = (1e-10,)
    out = {}
    for flags in ("1", "0"):
        monkeypatch.setenv("NPCG_LEVELFLAGS", flags)
        P = gnn.build_learned_batch(model, A, prob.rhs, values=vals)
        out[flags] = pcg.pcg_solve_batch(A, prob.rhs, P, pcg.SolveOptions(thresholds=thr, max_iter=3000), values=vals)
    (X, reps), (X0, reps0) = out["1"], out["0"]
    for s in range(64):
        assert reps[s].converged and reps0[s].converged
        assert abs(reps[s].iterations - reps0[s].iterations) <= 1, (s, reps[s].iterations, reps0[s].iterations)
        assert rel(X[:, s], X0[:, s]) <= X_TOL
    for s in (0, 2, 4):
        oA = port.Csr(A.n, A.row_ptr, A.col_idx, np.ascontiguousarray(vals[:, s]))
        oF = port.build_learned(ohp, model.params, oA, prob.rhs[:, s])
        ox, orep = port.pcg_solve(oA, prob.rhs[:, s], oF, thresholds=thr, max_iter=3000)
        assert orep.converged
        assert abs(reps[s].iterations - orep.iterations) <= 1, (s, reps[s].iterations, orep.iterations)
        assert rel(X[:, s], ox) <= X_TOL
