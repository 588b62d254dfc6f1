"""The device training step (csrc/train.cu through paper_2305_16432_b200.train)
against what pcgkit.train itself computed (tests/golden/train_*.npz) and
against the oracle's restatement at sizes the golden does not cover. fp64 on
both sides: the bars are summation-order bars (1e-10 relative), not fp32."""
import json
import os

import numpy as np
import pytest

from oracle import port, train_port
from paper_2305_16432_b200 import errors, gnn, inputs, sparse, train

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


class Tup:
    def __init__(self, A, b, x):
        self.A, self.b, self.x = A, b, x


def load(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    meta = json.loads(str(z["meta"]))
    names = [str(s) for s in z["param_names"]]
    params = {k: z["p_" + k].copy() for k in names}
    final = {k: z["q_" + k].copy() for k in names}
    tuples = []
    i = 0
    while f"t{i}_b" in z.files:
        A = sparse.SparseMatrixCsr(len(z[f"t{i}_b"]), z[f"t{i}_row_ptr"], z[f"t{i}_col_idx"], z[f"t{i}_values"])
        tuples.append(Tup(A, z[f"t{i}_b"], z[f"t{i}_x"]))
        i += 1
    hyper = gnn.GnnHyperParams(l=1, h=meta["h"], n_mp=meta["n_mp"], l_mp=1, h_mp=meta["h_mp"],
                               with_x0_head=meta["with_x0_head"])
    return z, meta, gnn.GnnModel(hyper, params), final, tuples


def close(got, want, rel):
    scale = max(np.abs(want).max(), 1e-300)
    return np.abs(got - want).max() <= rel * scale


@pytest.mark.parametrize("name", ["train_nohead", "train_x0head"])
def test_tuple_loss_and_gradients_match_pcgkit(gpu, name):
    z, meta, model, _, tuples = load(name)
    for i, t in enumerate(tuples):
        loss, grads = train.tuple_loss_and_grad(model, t.A, t.b, t.x, meta["x0_aux_weight"])
        want = float(z[f"t{i}_loss"])
        assert abs(loss - want) <= 1e-12 * max(1.0, abs(want))
        for k in model.params:
            assert close(grads[k], z[f"t{i}_g_{k}"], 1e-10), (i, k)


@pytest.mark.parametrize("name", ["train_nohead", "train_x0head"])
def test_training_run_matches_pcgkit(gpu, name, tmp_path):
    """train(): the permutation, minibatch means in tuple order, Adam, the
    final checkpoint and loss_curve.csv (train.py:229-284)."""
    z, meta, model, final, tuples = load(name)
    cfg = train.TrainConfig(loss_kind="data", learning_rate=meta["learning_rate"], batch_size=meta["batch_size"],
                            epochs=meta["epochs"], seed=meta["train_seed"], x0_aux_weight=meta["x0_aux_weight"],
                            checkpoint_every=2)
    before = {k: v.copy() for k, v in model.params.items()}
    trained, hist = train.train(model, tuples, cfg, out_dir=str(tmp_path))
    np.testing.assert_allclose([h["batch_loss"] for h in hist], z["train_losses"], rtol=1e-9)
    for k in final:
        np.testing.assert_allclose(trained.params[k], final[k], rtol=0, atol=1e-11 * max(1.0, np.abs(final[k]).max()))
        np.testing.assert_array_equal(model.params[k], before[k])  # the input model is not mutated
    assert [h["step"] for h in hist] == list(range(1, len(hist) + 1))
    assert sorted(os.listdir(tmp_path)) == ["checkpoint_000002.json", "checkpoint_000004.json",
                                            "checkpoint_000006.json", "loss_curve.csv", "model_final.json"]
    again = gnn.load_model(os.path.join(tmp_path, "model_final.json"))
    for k in final:
        np.testing.assert_array_equal(again.params[k], trained.params[k])


def test_gradients_latent64_vs_oracle(gpu):
    """Benchmark-shaped network (latent 64, 3 rounds) on a 24 x 24 heat
    problem: loss and gradients against the oracle's restatement; bitwise
    reproducible run to run."""
    old = gnn.FEATURE_WIDTH
    try:
        gnn.FEATURE_WIDTH = 64
        prob = inputs.heat_2d(k=24, cfg=7)
        A, b = prob.A, prob.rhs[:, 0]
        x = np.random.default_rng(3).standard_normal(A.n)
        hyper = gnn.GnnHyperParams(l=1, h=32, n_mp=3, l_mp=1, h_mp=64, with_x0_head=True)
        model = gnn.create_model(hyper, seed=5)
        for r in range(3):
            for s in ("node", "edge"):
                model.params[f"mp{r}.{s}.1.w"] *= 10.0
        loss, grads = train.tuple_loss_and_grad(model, A, b, x)
        loss2, grads2 = train.tuple_loss_and_grad(model, A, b, x)
        assert loss == loss2
        for k in grads:
            np.testing.assert_array_equal(grads[k], grads2[k])
        ohp = port.Hyper(l=1, h=32, n_mp=3, l_mp=1, h_mp=64, with_x0_head=True, width=64)
        oA = port.Csr(A.n, A.row_ptr, A.col_idx, A.values)
        oloss, ograds = train_port.tuple_loss_and_grad(ohp, model.params, oA, b, x)
        assert abs(loss - oloss) <= 1e-11 * abs(oloss)
        for k in model.params:
            assert close(grads[k], ograds[k], 1e-9), k
    finally:
        gnn.FEATURE_WIDTH = old


def test_apply_learned_factor_and_loss_data(gpu):
    prob = inputs.heat_2d(k=12, cfg=9)
    A, b = prob.A, prob.rhs[:, 0]
    rng = np.random.default_rng(1)
    low = A.strict_lower()
    lv = rng.uniform(-0.3, 0.3, low.nnz)
    x = rng.standard_normal(A.n)
    rows, cols = low.row_indices(), low.col_idx
    _, y = train_port.apply_factor(lv, rows, cols, A.diagonal(), x)
    got = train.apply_learned_factor(lv, A.diagonal(), x, A)
    assert close(got, y, 1e-13)
    want = float((y - b) @ (y - b))
    assert abs(train.loss_data(lv, A.diagonal(), x, b, A) - want) <= 1e-12 * want
    with pytest.raises(errors.DimensionMismatchError):
        train.apply_learned_factor(lv[:-1], A.diagonal(), x, A)
    with pytest.raises(errors.DimensionMismatchError):
        train.loss_data(lv, A.diagonal(), x, b[:-1], A)


def test_error_paths(gpu):
    import torch
    _, _, model, _, tuples = load("train_nohead")
    with pytest.raises(errors.DimensionMismatchError):
        train.train(model, [], train.TrainConfig())
    with pytest.raises(errors.DimensionMismatchError):
        train.TrainConfig(loss_kind="huber")
    with pytest.raises(NotImplementedError):
        train.train(model, tuples, train.TrainConfig(loss_kind="naive"))
    same, hist = train.train(model, tuples, train.TrainConfig(epochs=0))
    assert hist == [] and all(np.array_equal(same.params[k], model.params[k]) for k in model.params)
    tr = train.DeviceTrainer(model)
    g = tr.new_grad()
    g[3] = float("nan")
    before = tr.params()
    with pytest.raises(errors.NonFiniteGradientError):
        tr.adam_step(g, 1)
    after = tr.params()
    assert all(np.array_equal(before[k], after[k]) for k in before)  # no update on a bad gradient
    with pytest.raises(errors.DimensionMismatchError):
        tr.adam_step(torch.zeros_like(g), 0)
    ns = gnn.create_model(gnn.GnnHyperParams(l=1, h=8, n_mp=1, l_mp=1, h_mp=16, mode="north_star"), seed=0)
    with pytest.raises(errors.DimensionMismatchError):
        train.DeviceTrainer(ns)
