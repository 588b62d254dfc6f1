"""Golden training vectors produced by the REFERENCE itself (pcgkit.train).

Runs only in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba \
        python tests/golden/make_golden_train.py

For small seeded heat problems (this repo's inputs.heat_2d: matrices pinned
bitwise to pcgkit.fem by tests/test_inputs.py) the file records what
pcgkit.train computes: tuple_loss + ad.backward per tuple (loss and every
parameter's gradient, train.py:189-205), and a short train() run (batch
losses and final parameters, train.py:229-284, Adam train.py:164-185).
Two weight sets: without and with the x0 head (auxiliary loss term).
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from pcgkit import autodiff as ad, fem, gnn, sparse, train  # noqa: E402

from paper_2305_16432_b200 import inputs  # noqa: E402  (seeded matrices / loads only)


def tuples_for(count):
    out = []
    for j in range(count):
        prob = inputs.heat_2d(k=6 + j % 3, cfg=40 + j)
        A = sparse.SparseMatrixCsr(prob.A.n, prob.A.row_ptr, prob.A.col_idx, prob.A.values)
        b = prob.rhs[:, 0].copy()
        x = np.linalg.solve(A.to_dense(), b)
        out.append(fem.DatasetTuple(A, b, x, {"k": 6 + j % 3, "cfg": 40 + j}))
    return out


def main():
    for name, head in (("train_nohead", False), ("train_x0head", True)):
        gnn.FEATURE_WIDTH = 16
        hyper = gnn.GnnHyperParams(l=1, h=8, n_mp=2, l_mp=1, h_mp=16, with_x0_head=head)
        model = gnn.create_model(hyper, seed=11)
        for r in range(hyper.n_mp):  # non-trivial L' (the 0.1 processor gain cancelled)
            for s in ("node", "edge"):
                model.params[f"mp{r}.{s}.1.w"] *= 10.0
        tuples = tuples_for(5)
        rec = {"meta": json.dumps(dict(width=16, h=8, n_mp=2, h_mp=16, with_x0_head=head, seed=11,
                                       x0_aux_weight=0.1, batch_size=2, epochs=2, train_seed=3,
                                       learning_rate=1e-3))}
        names = sorted(model.params)
        rec["param_names"] = np.array(names)
        for nme in names:
            rec["p_" + nme] = model.params[nme]
        cfg = train.TrainConfig(loss_kind="data", learning_rate=1e-3, batch_size=2, epochs=2, seed=3)
        for i, t in enumerate(tuples):
            rec[f"t{i}_row_ptr"], rec[f"t{i}_col_idx"] = t.A.row_ptr, t.A.col_idx
            rec[f"t{i}_values"], rec[f"t{i}_b"], rec[f"t{i}_x"] = t.A.values, t.b, t.x
            graph = gnn.graph_from_system(t.A, t.b)
            loss, fwd = train.tuple_loss(model, graph, t, cfg)
            ad.backward(loss)
            rec[f"t{i}_loss"] = np.array(float(loss.value))
            for nme in names:
                g = fwd.param_tensors[nme].grad
                rec[f"t{i}_g_" + nme] = np.zeros_like(model.params[nme]) if g is None else g
        trained, hist = train.train(model, tuples, cfg)
        rec["train_losses"] = np.array([h["batch_loss"] for h in hist])
        for nme in names:
            rec["q_" + nme] = trained.params[nme]
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **rec)
        print(name, "losses", rec["train_losses"])


if __name__ == "__main__":
    main()
