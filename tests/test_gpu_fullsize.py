"""Parity at the benchmarked sizes, the oracle (oracle/port.py, pinned
bitwise to pcgkit) as the checker:

* config 2 in full (bench.py's workload: Poisson 256^2 jittered, n = 65,025,
  the latent-64 / 5-round GNN with the bench's weights, 64 GRF right-hand
  sides solved as one batch) -- L' within 1e-5 normwise, and for a spread of
  the 64 right-hand sides iterations within +-1 and x within 1e-8 of the
  oracle's fp64 solve (gnn.py:314-318 + pcg.py:75-176);
* config 3's real pattern (wave 512^2 without Dirichlet: 513 grid lines,
  n = 263,169) -- it must get a line-wavefront schedule (more than 512 lines,
  a 2- or 4-CTA cluster per system), apply_inverse bitwise against
  sparse.py:222-239, and two distinct systems end to end (per-system GNN at
  latent 64, rtol 1e-8) against the oracle.
"""
import numpy as np
import pytest

from oracle import port
from paper_2305_16432_b200 import _native, gnn, inputs, pcg, sparse

pytestmark = pytest.mark.gpu

L_TOL = 1e-5
X_TOL = 1e-8


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def seeded_model(monkeypatch, width=64, n_mp=5, h=64, seed=3, gain=10.0):
    """bench.py's weights: create_model(seed) with the processor output gain cancelled."""
    monkeypatch.setattr(gnn, "FEATURE_WIDTH", width)
    hyper = gnn.GnnHyperParams(l=1, h=h, n_mp=n_mp, l_mp=1, h_mp=h)
    model = gnn.create_model(hyper, seed=seed)
    for r in range(n_mp):
        for s in ("node", "edge"):
            model.params[f"mp{r}.{s}.1.w"] *= gain
    hp = port.Hyper(l=1, h=h, n_mp=n_mp, l_mp=1, h_mp=h, width=width)
    return model, hp


def ocsr(A, values=None):
    return port.Csr(A.n, A.row_ptr, A.col_idx, A.values if values is None else np.ascontiguousarray(values))


def line_info(A, batch):
    import ctypes
    out = [ctypes.c_int32() for _ in range(4)]
    _native.check(_native.lib().npcg_pattern_line_info(A.device_pattern().handle, *[ctypes.byref(o) for o in out],
                                                       batch))
    return [o.value for o in out]


def test_cfg2_full_size_trained_weights_vs_oracle(gpu, monkeypatch):
    """bench.py's default workload: config 2 with the committed trained
    checkpoint (weights/poisson2d_latent64_mp5.json, ~105 iterations). The
    same bars against the oracle's fp64 build_learned + pcg_solve."""
    import os

    import torch
    monkeypatch.setattr(gnn, "FEATURE_WIDTH", 64)
    path = os.path.join(os.path.dirname(os.path.abspath(gnn.__file__)), "weights", "poisson2d_latent64_mp5.json")
    model = gnn.load_model(path)
    hp = port.Hyper(l=1, h=model.hyper.h, n_mp=model.hyper.n_mp, l_mp=1, h_mp=model.hyper.h_mp, width=64)
    prob = inputs.poisson_2d(k=256, batch=64)
    A = prob.A
    P = gnn.build_learned(model, A, prob.rhs[:, 0])
    oA = ocsr(A)
    oF = port.build_learned(hp, model.params, oA, prob.rhs[:, 0])
    assert rel(P.factor.strict_lower.values, oF.lower.values) <= L_TOL
    opts = pcg.SolveOptions(thresholds=(1e-8,))
    X, reps = pcg.pcg_solve_batch(A, torch.from_numpy(prob.rhs).cuda(), P, opts)
    X = X.cpu().numpy()
    assert all(r.converged for r in reps)
    assert max(r.iterations for r in reps) < 200  # a trained preconditioner: Jacobi needs ~930, SGS ~330
    for s in (0, 13, 27, 40, 51, 63):
        ox, orep = port.pcg_solve(oA, prob.rhs[:, s], oF, thresholds=(1e-8,))
        assert orep.converged
        assert abs(reps[s].iterations - orep.iterations) <= 1, (s, reps[s].iterations, orep.iterations)
        assert rel(X[:, s], ox) <= X_TOL
        assert len(reps[s].history) == reps[s].iterations + 1


def test_cfg2_full_size_vs_oracle(gpu, monkeypatch):
    import torch
    prob = inputs.poisson_2d(k=256, batch=64)
    A = prob.A
    assert (A.n, A.nnz) == (65025, 453137)
    model, hp = seeded_model(monkeypatch)
    P = gnn.build_learned(model, A, prob.rhs[:, 0])
    oA = ocsr(A)
    oF = port.build_learned(hp, model.params, oA, prob.rhs[:, 0])
    assert rel(P.factor.strict_lower.values, oF.lower.values) <= L_TOL
    opts = pcg.SolveOptions(thresholds=(1e-8,))
    X, reps = pcg.pcg_solve_batch(A, torch.from_numpy(prob.rhs).cuda(), P, opts)
    X = X.cpu().numpy()
    for s in (0, 21, 42, 63):
        ox, orep = port.pcg_solve(oA, prob.rhs[:, s], oF, thresholds=(1e-8,))
        assert reps[s].converged and orep.converged
        assert abs(reps[s].iterations - orep.iterations) <= 1, (s, reps[s].iterations, orep.iterations)
        assert rel(X[:, s], ox) <= X_TOL
        assert len(reps[s].history) == reps[s].iterations + 1
    # decoupled from the GNN: the oracle's own L' through the device PCG
    Po = gnn.assemble_preconditioner(oF.lower.values, A)
    x, rep = pcg.pcg_solve(A, prob.rhs[:, 5], Po, opts)
    ox, orep = port.pcg_solve(oA, prob.rhs[:, 5], oF, thresholds=(1e-8,))
    assert abs(rep.iterations - orep.iterations) <= 1
    assert rel(x, ox) <= X_TOL
    h, ref = np.array(rep.history), np.array(orep.history)
    np.testing.assert_allclose(h[:4], ref[:4], rtol=1e-9)


@pytest.fixture(scope="module")
def cfg3():
    return inputs.wave_2d(k=512, batch=2)


def test_cfg3_pattern_takes_the_line_schedule(gpu, cfg3):
    A = cfg3.A
    assert A.n == 513 * 513
    lines, warps, steps, cluster = line_info(A, 32)
    assert lines == 513 and warps == 17 and steps == 2 * 513 - 1, (lines, warps, steps)
    assert cluster in (2, 4)


def test_cfg3_apply_inverse_bitwise(gpu, cfg3):
    A = cfg3.A
    rng = np.random.default_rng(5)
    low = A.strict_lower()
    vals = rng.uniform(-0.3, 0.3, size=low.nnz)
    F = sparse.LowerFactor(A.n, sparse.SparseMatrixCsr(A.n, low.row_ptr, low.col_idx, vals), A.diagonal())
    oF = port.Factor(A.n, port.Csr(A.n, low.row_ptr, low.col_idx, vals), A.diagonal())
    for _ in range(2):
        r = rng.standard_normal(A.n)
        np.testing.assert_array_equal(sparse.ldlt_apply_inverse(F, r), oF.apply_inverse(r))


def test_cfg3_two_distinct_systems_end_to_end(gpu, monkeypatch, cfg3):
    A, vals = cfg3.A, cfg3.values
    model, hp = seeded_model(monkeypatch)
    P = gnn.build_learned_batch(model, A, cfg3.rhs, values=vals)
    opts = pcg.SolveOptions(thresholds=(1e-8,))
    X, reps = pcg.pcg_solve_batch(A, cfg3.rhs, P, opts, values=vals)
    for s in range(2):
        oA = ocsr(A, vals[:, s])
        oF = port.build_learned(hp, model.params, oA, cfg3.rhs[:, s])
        assert rel(P.system_factor(s).strict_lower.values, oF.lower.values) <= L_TOL
        ox, orep = port.pcg_solve(oA, cfg3.rhs[:, s], oF, thresholds=(1e-8,))
        assert reps[s].converged and orep.converged
        assert abs(reps[s].iterations - orep.iterations) <= 1, (s, reps[s].iterations, orep.iterations)
        assert rel(X[:, s], ox) <= X_TOL


def test_cfg3_trained_checkpoint_end_to_end(gpu, monkeypatch, cfg3):
    """bench.py --config 3's default weights (weights/wave2d_latent64_mp5.json,
    ~11 iterations): one of the 513^2 systems end to end against the oracle."""
    import os
    monkeypatch.setattr(gnn, "FEATURE_WIDTH", 64)
    path = os.path.join(os.path.dirname(os.path.abspath(gnn.__file__)), "weights", "wave2d_latent64_mp5.json")
    model = gnn.load_model(path)
    hp = port.Hyper(l=1, h=model.hyper.h, n_mp=model.hyper.n_mp, l_mp=1, h_mp=model.hyper.h_mp, width=64)
    A, vals = cfg3.A, cfg3.values
    P = gnn.build_learned_batch(model, A, cfg3.rhs, values=vals)
    X, reps = pcg.pcg_solve_batch(A, cfg3.rhs, P, pcg.SolveOptions(thresholds=(1e-8,)), values=vals)
    assert all(r.converged for r in reps) and max(r.iterations for r in reps) < 20  # Jacobi needs ~22
    s = 1
    oA = ocsr(A, vals[:, s])
    oF = port.build_learned(hp, model.params, oA, cfg3.rhs[:, s])
    assert rel(P.system_factor(s).strict_lower.values, oF.lower.values) <= L_TOL
    ox, orep = port.pcg_solve(oA, cfg3.rhs[:, s], oF, thresholds=(1e-8,))
    assert orep.converged
    assert abs(reps[s].iterations - orep.iterations) <= 1, (reps[s].iterations, orep.iterations)
    assert rel(X[:, s], ox) <= X_TOL
