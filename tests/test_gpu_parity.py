"""End-to-end GPU parity against the reference's own outputs (goldens from
tests/golden/make_golden.py) and the pinned oracle.

Bars (BASELINE.json north_star):
  L' (fp32 GNN)   normwise relative error <= 1e-5
  iterations      within +-1 of the reference
  x               within 1e-8 relative (2-norm) of the reference's fp64 x
Kernel-level probes are bitwise (sparse.py:213-239 arithmetic contract).
History: the first iterations of a solve with the reference's own L' must
agree to ~1e-12 (only reduction order differs); afterwards CG amplifies
rounding, so the whole trace is held to an envelope.
"""
import numpy as np
import pytest

from golden_util import GOLDEN, Golden
from oracle import port
from paper_2305_16432_b200 import gnn, pcg, sparse

pytestmark = pytest.mark.gpu

L_TOL = 1e-5
X_TOL = 1e-8


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def model_for(g: Golden, monkeypatch):
    m = g.meta
    if m["weights"] == "trained":
        return gnn.load_model(f"{GOLDEN}/{m['checkpoint']}")
    monkeypatch.setattr(gnn, "FEATURE_WIDTH", m["width"])
    hyper = gnn.GnnHyperParams(**g.hyper_kwargs())
    model = gnn.create_model(hyper, seed=m["seed"])
    for r in range(hyper.n_mp):
        for s in ("node", "edge"):
            model.params[f"mp{r}.{s}.1.w"] *= 10.0
    return model


def matrix(g: Golden, values=None):
    return sparse.SparseMatrixCsr(g.n, g.row_ptr, g.col_idx, g.values if values is None else values)


@pytest.mark.parametrize("name", ["cfg1_trained", "cfg1_perturbed"])
def test_probes_bitwise(gpu, name):
    g = Golden(name)
    c = g.case(0)
    A = matrix(g)
    np.testing.assert_array_equal(sparse.spmv(A, c["probe_r"]), c["probe_Ar"])
    P = gnn.assemble_preconditioner(c["lower"], A)
    np.testing.assert_array_equal(P.apply_inverse(c["probe_r"]), c["probe_z"])


@pytest.mark.parametrize("name", ["cfg1_trained", "cfg1_perturbed"])
def test_single_system_end_to_end(gpu, monkeypatch, name):
    g = Golden(name)
    c = g.case(0)
    A, b = matrix(g), g.rhs[:, 0]
    model = model_for(g, monkeypatch)
    # GNN outputs
    graph = gnn.graph_from_system(A, b)
    M, x0 = gnn.run(model, graph)
    assert rel(M, c["M"]) <= L_TOL
    if c["x0"].size:
        assert rel(x0, c["x0"]) <= L_TOL
    P = gnn.build_learned(model, A, b)
    assert P.kind == "learned"
    assert rel(P.factor.strict_lower.values, c["lower"]) <= L_TOL
    np.testing.assert_array_equal(P.factor.diag, A.diagonal())
    thr = tuple(g.meta["thresholds"])
    x, rep = pcg.pcg_solve(A, b, P, pcg.SolveOptions(thresholds=thr, max_iter=g.meta["max_iter"]))
    assert rep.converged == bool(c["converged"])
    assert abs(rep.iterations - int(c["iterations"])) <= 1
    assert rel(x, c["x"]) <= X_TOL
    assert len(rep.history) == rep.iterations + 1
    # all default thresholds
    _, rep_all = pcg.pcg_solve(A, b, P, pcg.SolveOptions(max_iter=g.meta["max_iter"]))
    got = [rep_all.iterations_to.get(t, -1) for t in pcg.DEFAULT_THRESHOLDS]
    assert np.all(np.abs(np.array(got) - c["all_iterations_to"]) <= 1), (got, c["all_iterations_to"])


@pytest.mark.parametrize("name", ["cfg1_trained", "cfg1_perturbed"])
def test_history_with_reference_factor(gpu, name):
    """Decoupled from the GNN: PCG on the reference's own L'."""
    g = Golden(name)
    c = g.case(0)
    A, b = matrix(g), g.rhs[:, 0]
    P = gnn.assemble_preconditioner(c["lower"], A)
    thr = tuple(g.meta["thresholds"])
    x, rep = pcg.pcg_solve(A, b, P, pcg.SolveOptions(thresholds=thr, max_iter=g.meta["max_iter"]))
    h, ref = np.array(rep.history), c["history"]
    assert abs(len(h) - len(ref)) <= 1
    k = min(4, len(h), len(ref))
    np.testing.assert_allclose(h[:k], ref[:k], rtol=1e-12)
    m = min(len(h), len(ref))
    # envelope of the whole trace (CG residual norms jump transiently
    # under a mere change of summation order -- it measured 0.11 decades at k = 42 on this
    # shape). Measured here (tools/history_envelope.py): 6e-15 on the trained golden, 0.098
    # on the perturbed one; the bars leave a factor ~2.5 over that.
    bar = 1e-6 if name == "cfg1_trained" else 0.25
    assert np.max(np.abs(np.log10(h[:m] / ref[:m]))) <= bar
    assert rel(x, c["x"]) <= X_TOL


def test_multi_rhs_shared_factor_latent64(gpu, monkeypatch):
    """Config-2 shape: one L' (GNN at latent 64 on RHS 0), B right-hand sides."""
    g = Golden("cfg2_small_f64")
    A = matrix(g)
    model = model_for(g, monkeypatch)
    P = gnn.build_learned(model, A, g.rhs[:, 0])
    assert rel(P.factor.strict_lower.values, g.z["lower"]) <= L_TOL
    thr = tuple(g.meta["thresholds"])
    X, reps = pcg.pcg_solve_batch(A, g.rhs, P, pcg.SolveOptions(thresholds=thr))
    for s, rep in enumerate(reps):
        c = g.case(s)
        assert rep.converged
        assert abs(rep.iterations - int(c["iterations"])) <= 1, (s, rep.iterations, c["iterations"])
        assert rel(X[:, s], c["x"]) <= X_TOL
    # a batched solve agrees with the single-RHS solve (reductions are
    # partitioned differently, so agreement is to rounding, not bitwise)
    x0, rep0 = pcg.pcg_solve(A, g.rhs[:, 0], P, pcg.SolveOptions(thresholds=thr))
    assert abs(rep0.iterations - reps[0].iterations) <= 1
    assert rel(x0, X[:, 0]) <= X_TOL


def test_distinct_systems_batch_latent64(gpu, monkeypatch):
    """Config-3 shape: B distinct matrices on one pattern, one GNN per system."""
    g = Golden("cfg3_small_f64")
    vals = g.z["values_batch"]
    A = matrix(g, np.ascontiguousarray(vals[:, 0]))
    model = model_for(g, monkeypatch)
    P = gnn.build_learned_batch(model, A, g.rhs, values=vals)
    assert P.batch == vals.shape[1]
    thr = tuple(g.meta["thresholds"])
    X, reps = pcg.pcg_solve_batch(A, g.rhs, P, pcg.SolveOptions(thresholds=thr), values=vals)
    for s, rep in enumerate(reps):
        c = g.case(s)
        assert rel(P.system_factor(s).strict_lower.values, c["lower"]) <= L_TOL
        assert abs(rep.iterations - int(c["iterations"])) <= 1
        assert rel(X[:, s], c["x"]) <= X_TOL


def test_gpu_matches_oracle_on_fresh_seeds(gpu):
    """Beyond the goldens: random perturbed F=16 weights, oracle as checker."""
    from paper_2305_16432_b200 import inputs
    prob = inputs.heat_2d(k=20, cfg=11)
    A, b = prob.A, prob.rhs[:, 0]
    oA = port.Csr(A.n, A.row_ptr, A.col_idx, A.values)
    for seed in (1, 2):
        hyper = gnn.GnnHyperParams(l=1, h=16, n_mp=2, l_mp=1, h_mp=16)
        model = gnn.create_model(hyper, seed=seed)
        for k in list(model.params):
            if k.endswith(".b"):
                model.params[k] = np.random.default_rng(seed).normal(0, 0.25, model.params[k].shape)
        P = gnn.build_learned(model, A, b)
        oF = port.build_learned(port.Hyper(l=1, h=16, n_mp=2, l_mp=1, h_mp=16), model.params, oA, b)
        assert rel(P.factor.strict_lower.values, oF.lower.values) <= L_TOL
        x, rep = pcg.pcg_solve(A, b, P, pcg.SolveOptions(thresholds=(1e-10,), max_iter=3000))
        ox, orep = port.pcg_solve(oA, b, oF, thresholds=(1e-10,), max_iter=3000)
        assert rep.converged == orep.converged
        assert abs(rep.iterations - orep.iterations) <= 1
        assert rel(x, ox) <= X_TOL
