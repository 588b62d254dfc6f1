"""Preconditioners in the common LDL^T form (mirrors pcgkit.preconditioners,
/root/reference/pkg/src/pcgkit/preconditioners.py:1-222).

``FactorPreconditioner`` is the object ``pcg_solve`` consumes. Its factor
lives on the device as (pattern, S, D): S carries L' on both triangles of a
symmetric pattern, D the diagonal; a batch of B factors on one pattern is a
single object (``batch`` > 1). The host ``LowerFactor`` view is produced on
demand. Only the classic builders that reuse the same kernels are provided
(identity, Jacobi, symmetric Gauss-Seidel); IC(0)/IC(2) are out of scope
(SURVEY.md section 2).
"""
from __future__ import annotations

import numpy as np

from . import _native
from .errors import NotSpdError
from .sparse import (LowerFactor, SparseMatrixCsr, apply_inverse_device, is_device, to_device,
                     _torch)

VALID_KINDS = frozenset({"identity", "jacobi", "gauss_seidel", "ic0", "ic2", "learned"})


class FactorPreconditioner:
    """P = (I+L) D (I+L)^T with its construction tag (preconditioners.py:31-50)."""

    def __init__(self, kind, factor: LowerFactor | None = None, *, device=None, lower_pattern=None):
        if kind not in VALID_KINDS:
            raise ValueError(f"unknown preconditioner kind {kind!r}")
        if factor is None and device is None:
            raise ValueError("need a host factor or a device factor")
        self.kind = kind
        self._factor = factor
        # device = (pattern, S, s_batched, D, d_batched, B, n)
        self._device = device
        self._lower_pattern = lower_pattern  # SparseMatrixCsr strict-lower pattern (learned path)

    # -- reference surface ----------------------------------------------------------

    @property
    def batch(self) -> int:
        return 1 if self._device is None else self._device[5]

    @property
    def n(self) -> int:
        return self._factor.n if self._factor is not None else self._device[6]

    @property
    def factor(self) -> LowerFactor:
        """Host LowerFactor (system 0 of a batch); copied back on first use."""
        if self._factor is None:
            self._factor = self.system_factor(0)
        return self._factor

    def system_factor(self, b: int) -> LowerFactor:
        torch = _torch()
        pat, S, sb, D, db, B, n = self._device
        lp = self._lower_pattern
        m = lp.nnz
        low = torch.empty(max(m * B, 1), dtype=torch.float64, device="cuda")
        if m:
            _native.check(_native.lib().npcg_factor_to_lower(pat.handle, B if sb else 1, _native.ptr(S),
                                                             _native.ptr(low), _native.stream_handle()))
        vals = low[: m * (B if sb else 1)].view(m, B if sb else 1)[:, b if sb else 0]
        d = D.view(n, B if db else 1)[:, b if db else 0]
        sl = SparseMatrixCsr(n, lp.row_ptr, lp.col_idx, vals.cpu().numpy())
        return LowerFactor(n, sl, d.cpu().numpy())

    def device_factor(self):
        """(pattern, S, s_batched, D, d_batched, B) for the device PCG loop."""
        if self._device is None:
            pat, S, D = self._factor.device()
            self._device = (pat, S, False, D, False, 1, self._factor.n)
        return self._device[:6]

    def apply_inverse(self, r):
        """z = P^{-1} r on the device (sparse.py:265-275); r is (n,) or (n, B)."""
        on_dev = is_device(r)
        pat, S, sb, D, db, B = self.device_factor()
        rd = to_device(r)
        cols = 1 if rd.dim() == 1 else rd.shape[1]
        if rd.shape[0] != self.n or (B > 1 and cols != B):
            from .errors import DimensionMismatchError
            raise DimensionMismatchError(f"rhs has shape {tuple(r.shape)}, expected ({self.n},)")
        z = apply_inverse_device(pat, S, sb, D, db, rd, cols)
        return z if on_dev else z.cpu().numpy()

    def to_dense(self) -> np.ndarray:
        return self.factor.to_dense()


def _empty_strict_lower(n: int) -> SparseMatrixCsr:
    return SparseMatrixCsr(n, np.zeros(n + 1, dtype=np.int64), np.empty(0, dtype=np.int64), np.empty(0))


def _positive_diagonal(A: SparseMatrixCsr) -> np.ndarray:
    d = A.diagonal()
    if np.any(d <= 0.0):
        bad = int(np.argmax(d <= 0.0))
        raise NotSpdError(f"nonpositive diagonal entry at row {bad}", pivot=bad)
    return d


def identity_preconditioner(n: int) -> FactorPreconditioner:
    return FactorPreconditioner("identity", LowerFactor(n, _empty_strict_lower(n), np.ones(n)))


def build_jacobi(A: SparseMatrixCsr) -> FactorPreconditioner:
    """P = diag(A) (preconditioners.py:70-73)."""
    d = _positive_diagonal(A)
    return FactorPreconditioner("jacobi", LowerFactor(A.n, _empty_strict_lower(A.n), d.copy()))


def build_gauss_seidel(A: SparseMatrixCsr) -> FactorPreconditioner:
    """Symmetric Gauss-Seidel, L = L_A D^-1 (preconditioners.py:76-85)."""
    d = _positive_diagonal(A)
    low = A.strict_lower()
    scaled = SparseMatrixCsr(A.n, low.row_ptr, low.col_idx, low.values / d[low.col_idx])
    return FactorPreconditioner("gauss_seidel", LowerFactor(A.n, scaled, d.copy()))


BUILDERS = {"jacobi": build_jacobi, "gauss_seidel": build_gauss_seidel}


def build(kind: str, A: SparseMatrixCsr) -> FactorPreconditioner:
    if kind == "identity":
        return identity_preconditioner(A.n)
    try:
        return BUILDERS[kind](A)
    except KeyError:
        raise ValueError(f"no builder for preconditioner kind {kind!r}") from None
