"""Data loss, end-to-end gradients, Adam and the training loop on the device.

Mirror of the reference's ``pcgkit.train`` for the matrix-free data loss
``loss_data = ||(I+L') D (I+L')^T x - b||^2`` (train.py:104-150): the
network forward, symmetrisation, the factor application, the whole reverse
pass (what ``ad.backward`` does with the tape, autodiff.py:113-253) and Adam
(train.py:164-185) run in ``libnpcg`` (csrc/train.cu, fp64 like the
reference). Same names, argument meaning and errors as the reference;
what is NOT covered: ``loss_kind="naive"`` (its gradient is a dense O(n^2)
oracle in the reference, train.py:66-100) and the north_star network
extensions (no reference to train against).
"""
from __future__ import annotations

import csv
import ctypes
import logging
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native, gnn
from .errors import DimensionMismatchError, DivergenceError, NonFiniteGradientError
from .sparse import LowerFactor, SparseMatrixCsr, ldlt_apply, to_device

log = logging.getLogger(__name__)


@dataclass(frozen=True)
class TrainConfig:
    """train.py:37-52."""
    loss_kind: str = "data"  # "data" (device) or "naive" (not on the device path)
    learning_rate: float = 1e-3
    batch_size: int = 16
    epochs: int = 1
    seed: int = 0
    checkpoint_every: int = 0  # steps between checkpoints; 0 = final only
    x0_aux_weight: float = 0.1  # weight of the x0-head regression term

    def __post_init__(self):
        if self.loss_kind not in ("data", "naive"):
            raise DimensionMismatchError(f"unknown loss kind {self.loss_kind!r}")
        if self.learning_rate <= 0 or self.batch_size < 1 or self.epochs < 0:
            raise DimensionMismatchError("bad training configuration")


# ---------------------------------------------------------------------------
# losses (train.py:104-150)
# ---------------------------------------------------------------------------


def _lower_factor(lower_values, diag, A: SparseMatrixCsr) -> LowerFactor:
    pattern = A.strict_lower()
    lower_values = np.asarray(lower_values, dtype=np.float64)
    if lower_values.shape != (pattern.nnz,):
        raise DimensionMismatchError(f"expected {pattern.nnz} lower values, got {lower_values.shape}")
    diag = np.asarray(diag, dtype=np.float64)
    if diag.shape != (A.n,):
        raise DimensionMismatchError("x and diag must have one entry per row")
    return LowerFactor(A.n, SparseMatrixCsr(A.n, pattern.row_ptr, pattern.col_idx, lower_values), diag)


def apply_learned_factor(lower_values, diag, x, A: SparseMatrixCsr):
    """y = (I+L') D (I+L')^T x without forming the product (train.py:104-141),
    as three device products."""
    x = np.asarray(x, dtype=np.float64)
    if x.shape != (A.n,):
        raise DimensionMismatchError("x and diag must have one entry per row")
    return ldlt_apply(_lower_factor(lower_values, diag, A), x)


def loss_data(lower_values, diag, x, b, A: SparseMatrixCsr) -> float:
    """||(I+L') D (I+L')^T x - b||_2^2, matrix-free (train.py:143-152)."""
    b = np.asarray(b, dtype=np.float64)
    if b.shape != (A.n,):
        raise DimensionMismatchError("b must have one entry per row")
    r = apply_learned_factor(lower_values, diag, x, A) - b
    return float(r @ r)


# ---------------------------------------------------------------------------
# device trainer
# ---------------------------------------------------------------------------


class DeviceTrainer:
    """Weights, Adam moments and workspace of one model on the device
    (``npcg_trainer``). ``tuple_grad`` is tuple_loss + ad.backward
    (train.py:189-205), ``adam_step`` is train.py:164-185."""

    def __init__(self, model: gnn.GnnModel):
        gnn._validate_params(model, model.width)
        hp = model.hyper
        if hp.north_star:
            raise DimensionMismatchError("the device training step covers the reference network only")
        self.hyper, self.width = hp, model.width
        self._specs = gnn._layer_specs(hp, model.width)
        self._lib = _native.lib()
        blob = model._blob()
        d = _native.GnnDesc(model.width, hp.h, hp.l, hp.h_mp, hp.l_mp, hp.n_mp, int(hp.normalize),
                            int(hp.with_x0_head), 0, hp.dim)
        h = ctypes.c_void_p()
        _native.check(self._lib.npcg_trainer_create(ctypes.byref(d), blob.ctypes.data, len(blob), ctypes.byref(h)))
        self._h = h
        self.n_weights = len(blob)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.npcg_trainer_destroy(h)
            self._h = None

    # -- parameter blob <-> dict (the checkpoint layout of GnnModel._blob) ----------
    def unpack(self, blob) -> dict:
        out, off = {}, 0
        for name, fi, fo in self._specs:
            out[name + ".w"] = np.array(blob[off: off + fi * fo]).reshape(fi, fo)
            off += fi * fo
            out[name + ".b"] = np.array(blob[off: off + fo])
            off += fo
        return out

    def params(self) -> dict:
        blob = np.empty(self.n_weights)
        _native.check(self._lib.npcg_trainer_get_weights(self._h, blob.ctypes.data))
        return self.unpack(blob)

    def new_grad(self):
        import torch
        return torch.zeros(self.n_weights, dtype=torch.float64, device="cuda")

    def tuple_grad(self, A: SparseMatrixCsr, b, x, grad_accum, x0_aux_weight: float = 0.1) -> float:
        """Loss of one tuple; its parameter gradient is added to
        ``grad_accum`` (a ``new_grad()`` tensor)."""
        b = np.asarray(b, dtype=np.float64)
        x = np.asarray(x, dtype=np.float64)
        if b.shape != (A.n,) or x.shape != (A.n,):
            raise DimensionMismatchError("b and x must have one entry per row")
        gnn._check_graph_system(A)
        node_in, edge_in = b, A.values
        if self.hyper.normalize:  # gnn.py:239-245, the reference's sorted statistics
            mu, sd = gnn._sorted_stats(b)
            node_in = (b - mu) / sd
            mu, sd = gnn._sorted_stats(A.values)
            edge_in = (A.values - mu) / sd
        pat = A.device_pattern(factor=True)
        loss = ctypes.c_double()
        bd, xd, nd, ed = to_device(b), to_device(x), to_device(node_in), to_device(edge_in)
        _native.check(self._lib.npcg_trainer_tuple_grad(
            self._h, pat.handle, _native.ptr(A.device_values()), _native.ptr(nd), _native.ptr(ed), _native.ptr(bd),
            _native.ptr(xd), float(x0_aux_weight), ctypes.byref(loss), _native.ptr(grad_accum),
            _native.stream_handle()))
        return float(loss.value)

    def adam_step(self, grad, t: int, learning_rate: float = 1e-3, beta1: float = 0.9, beta2: float = 0.999,
                  eps: float = 1e-8, grad_scale: float = 1.0) -> None:
        if t < 1:
            raise DimensionMismatchError("Adam step index starts at 1")
        bad = ctypes.c_int32()
        _native.check(self._lib.npcg_trainer_adam_step(self._h, _native.ptr(grad), float(grad_scale), int(t),
                                                       float(learning_rate), float(beta1), float(beta2), float(eps),
                                                       ctypes.byref(bad), _native.stream_handle()))
        if bad.value:
            raise NonFiniteGradientError("non-finite gradient")


def batch_gradients(trainer: DeviceTrainer, tuples, indices, config: TrainConfig):
    """Mean loss and the SUM of parameter gradients (device tensor) over one
    minibatch, accumulated in tuple-index order (train.py:208-226); the mean
    is taken by adam_step's ``grad_scale = 1 / len(indices)``."""
    grad = trainer.new_grad()
    total = 0.0
    for i in indices:
        t = tuples[i]
        total += trainer.tuple_grad(t.A, t.b, t.x, grad, config.x0_aux_weight)
    return total * (1.0 / len(indices)), grad


def tuple_loss_and_grad(model: gnn.GnnModel, A: SparseMatrixCsr, b, x, x0_aux_weight: float = 0.1):
    """(loss, {name: gradient}) of one tuple: train.tuple_loss followed by
    ad.backward, as plain arrays."""
    tr = DeviceTrainer(model)
    grad = tr.new_grad()
    loss = tr.tuple_grad(A, b, x, grad, x0_aux_weight)
    return loss, tr.unpack(grad.cpu().numpy())


# ---------------------------------------------------------------------------
# training loop (train.py:229-284)
# ---------------------------------------------------------------------------


def train(model: gnn.GnnModel, tuples, config: TrainConfig, out_dir=None):
    """Minibatch Adam over (A, b, x) tuples; returns (model, loss history).

    The input model is not mutated. History rows are dicts with step, epoch,
    batch_loss and wall_seconds; when ``out_dir`` is given they are also
    written to loss_curve.csv next to the checkpoints. Training aborts with
    DivergenceError if a batch loss exceeds 1e6 x the initial batch loss."""
    if not tuples:
        raise DimensionMismatchError("empty training set")
    if config.loss_kind != "data":
        raise NotImplementedError("the device training path implements loss_kind='data' (the naive loss's "
                                  "gradient is a dense oracle in the reference, train.py:66-100)")
    model = model.copy()
    if config.epochs == 0:
        return model, []
    trainer = DeviceTrainer(model)
    rng = np.random.default_rng(config.seed)
    history = []
    guard_level = None
    step = 0
    started = time.perf_counter()
    if out_dir is not None:
        os.makedirs(out_dir, exist_ok=True)

    def snapshot():
        return gnn.GnnModel(model.hyper, trainer.params())

    for epoch in range(config.epochs):
        order = rng.permutation(len(tuples))
        for lo in range(0, len(order), config.batch_size):
            batch = order[lo: lo + config.batch_size]
            loss, grad = batch_gradients(trainer, tuples, batch, config)
            if guard_level is None:
                guard_level = 1e6 * max(loss, 1e-300)
            elif loss > guard_level:
                raise DivergenceError(f"batch loss {loss:.3e} exceeds 1e6 x initial at step {step}")
            step += 1
            trainer.adam_step(grad, step, config.learning_rate, grad_scale=1.0 / len(batch))
            history.append({"step": step, "epoch": epoch, "batch_loss": loss,
                            "wall_seconds": time.perf_counter() - started})
            if out_dir is not None and config.checkpoint_every and step % config.checkpoint_every == 0:
                gnn.save_model(os.path.join(out_dir, f"checkpoint_{step:06d}.json"), snapshot())
        log.info("epoch %d done: last batch loss %.6e", epoch, history[-1]["batch_loss"])
    trained = snapshot()
    if out_dir is not None:
        gnn.save_model(os.path.join(out_dir, "model_final.json"), trained)
        write_loss_curve(os.path.join(out_dir, "loss_curve.csv"), history)
    return trained, history


def write_loss_curve(path, history) -> None:
    with open(path, "w", encoding="ascii", newline="") as fh:
        writer = csv.DictWriter(fh, fieldnames=["step", "epoch", "batch_loss", "wall_seconds"])
        writer.writeheader()
        writer.writerows(history)
