"""The oracle's training restatement (oracle/train_port.py) against what
pcgkit.train itself computed (tests/golden/train_*.npz, made by
tests/golden/make_golden_train.py): per-tuple loss and every parameter
gradient (train.py:189-205 + ad.backward), the minibatch mean, Adam and a
short training run (train.py:164-185, 229-284)."""
import json
import os

import numpy as np
import pytest

from oracle import port, train_port

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    meta = json.loads(str(z["meta"]))
    names = [str(s) for s in z["param_names"]]
    params = {k: z["p_" + k].copy() for k in names}
    final = {k: z["q_" + k].copy() for k in names}
    tuples = []
    i = 0
    while f"t{i}_b" in z.files:
        A = port.Csr(len(z[f"t{i}_b"]), z[f"t{i}_row_ptr"], z[f"t{i}_col_idx"], z[f"t{i}_values"])
        tuples.append((A, z[f"t{i}_b"], z[f"t{i}_x"]))
        i += 1
    hp = port.Hyper(l=1, h=meta["h"], n_mp=meta["n_mp"], l_mp=1, h_mp=meta["h_mp"],
                    with_x0_head=meta["with_x0_head"], width=meta["width"])
    return z, meta, hp, params, final, tuples


@pytest.mark.parametrize("name", ["train_nohead", "train_x0head"])
def test_tuple_loss_and_gradients_match_pcgkit(name):
    z, meta, hp, params, _, tuples = load(name)
    for i, (A, b, x) in enumerate(tuples):
        loss, grads = train_port.tuple_loss_and_grad(hp, params, A, b, x, meta["x0_aux_weight"])
        assert abs(loss - float(z[f"t{i}_loss"])) <= 1e-13 * max(1.0, abs(loss))
        for k in params:
            want = z[f"t{i}_g_{k}"]
            got = np.zeros_like(want) if grads[k] is None else grads[k]
            scale = max(np.abs(want).max(), 1e-300)
            assert np.abs(got - want).max() <= 1e-11 * scale, (i, k)


@pytest.mark.parametrize("name", ["train_nohead", "train_x0head"])
def test_training_run_matches_pcgkit(name):
    z, meta, hp, params, final, tuples = load(name)
    got, losses = train_port.train(hp, params, tuples, batch_size=meta["batch_size"], epochs=meta["epochs"],
                                   seed=meta["train_seed"], learning_rate=meta["learning_rate"],
                                   x0_aux_weight=meta["x0_aux_weight"])
    np.testing.assert_allclose(losses, z["train_losses"], rtol=1e-10)
    for k in params:
        np.testing.assert_allclose(got[k], final[k], rtol=0, atol=1e-12 * max(1.0, np.abs(final[k]).max()))
