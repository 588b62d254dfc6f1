"""north_star GNN mode, host side (no GPU): the numpy restatement
(oracle/port.py) is the mode's only oracle -- with the extensions off it is
the pinned reference path itself (tests/test_oracle_golden.py); here its
parameter set matches the package's, the exp-diagonal factor is exactly
P = L L^T, and checkpoints round-trip."""
import numpy as np
import pytest

from oracle import port
from paper_2305_16432_b200 import gnn, inputs
from paper_2305_16432_b200.errors import DataFormatError, DimensionMismatchError


def test_parameters_match_the_oracle(monkeypatch):
    monkeypatch.setattr(gnn, "FEATURE_WIDTH", 16)
    for dim in (2, 3):
        hyper = gnn.GnnHyperParams(l=1, h=16, n_mp=3, l_mp=1, h_mp=16, mode="north_star", dim=dim)
        model = gnn.create_model(hyper, seed=4)
        hp = port.Hyper(l=1, h=16, n_mp=3, l_mp=1, h_mp=16, width=16, mode="north_star", dim=dim)
        ref = port.create_params(hp, 4)
        assert sorted(model.params) == sorted(ref)
        for k in ref:
            np.testing.assert_array_equal(model.params[k], ref[k])
        assert model.params["edge_enc.0.w"].shape == (2 + dim, 16)
        assert model.params["node_enc.0.w"].shape == (2, 16)
    # the reference network draws are untouched by the mode's existence
    r = gnn.create_model(gnn.GnnHyperParams(l=1, h=16, n_mp=3, l_mp=1, h_mp=16), seed=4)
    assert not any(k.endswith(".ln.g") for k in r.params)


def test_exp_factor_is_l_lt():
    prob = inputs.heat_2d(k=6)
    A = prob.A
    oA = port.Csr(A.n, A.row_ptr, A.col_idx, A.values)
    hp = port.Hyper(l=1, h=8, n_mp=2, l_mp=1, h_mp=8, width=16, mode="north_star", dim=2)
    params = port.create_params(hp, 1)
    F = port.build_learned(hp, params, oA, prob.rhs[:, 0], mesh=prob.geometry)
    # rebuild L from the network outputs and compare P = L L^T with U D U^T
    g = port.graph_from_system(oA, prob.rhs[:, 0])
    g.node_in, g.edge_in = port.north_star_inputs(g, prob.rhs[:, 0], oA, *prob.geometry)
    M, _ = port.gnn_run(hp, params, g)
    L = np.zeros((A.n, A.n))
    for p in range(A.nnz):
        i, j = g.src[p], g.dst[p]
        if i == j:
            L[i, i] = np.exp(M[p])
        elif i > j:
            L[i, j] = 0.5 * (M[p] + M[g.pair[p]])
    scale = np.abs(L @ L.T).max()
    np.testing.assert_allclose(F.dense(), L @ L.T, rtol=0, atol=1e-13 * scale)
    L2 = (np.eye(A.n) + F.lower.dense()) * np.sqrt(F.diag)  # (I + U) D^1/2 is L itself
    np.testing.assert_allclose(L2, L, rtol=1e-15, atol=1e-15)


def test_checkpoint_roundtrip(tmp_path, monkeypatch):
    monkeypatch.setattr(gnn, "FEATURE_WIDTH", 16)
    hyper = gnn.GnnHyperParams(l=1, h=8, n_mp=2, l_mp=1, h_mp=8, mode="north_star", dim=3)
    model = gnn.create_model(hyper, seed=2)
    model.params["mp1.edge.ln.g"] = model.params["mp1.edge.ln.g"] * 1.5
    path = tmp_path / "ns.json"
    gnn.save_model(path, model)
    assert '"format_version": 2' in path.read_text()
    back = gnn.load_model(path)
    assert back.hyper == hyper
    for k in model.params:
        np.testing.assert_array_equal(back.params[k], model.params[k])
    ref = gnn.create_model(gnn.GnnHyperParams(l=1, h=8, n_mp=2, l_mp=1, h_mp=8), seed=2)
    gnn.save_model(tmp_path / "ref.json", ref)
    assert '"format_version": 1' in (tmp_path / "ref.json").read_text()
    bad = (tmp_path / "ref.json").read_text().replace('"h": 8,', '"dim": 3, "h": 8,', 1)
    (tmp_path / "bad.json").write_text(bad)
    with pytest.raises(DataFormatError):
        gnn.load_model(tmp_path / "bad.json")


def test_mode_validation():
    with pytest.raises(DimensionMismatchError):
        gnn.GnnHyperParams(mode="mystery")
    with pytest.raises(DimensionMismatchError):
        gnn.GnnHyperParams(mode="north_star", dim=4)


@pytest.mark.parametrize("make", [lambda: inputs.heat_2d(k=5), lambda: inputs.poisson_2d(k=6, batch=1),
                                  lambda: inputs.poisson_3d(k=4, batch=1)])
def test_geometry_rows(make):
    prob = make()
    pos, flag = prob.geometry
    assert pos.shape[0] == prob.A.n and flag.shape == (prob.A.n,)
    assert flag.any() and not flag.all()
