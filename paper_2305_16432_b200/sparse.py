"""CSR storage, device patterns, SpMV and LDL^T factor application.

Mirrors ``pcgkit.sparse`` (/root/reference/pkg/src/pcgkit/sparse.py): same
class names, fields, invariants and errors. Storage stays host-side numpy
(int64 indices, float64 values) exactly as in the reference so existing
callers build matrices the same way; the first compute call uploads the
pattern once (``DevicePattern``, analysed by libnpcg) and the values, and
every product / solve runs as sm_100a kernels. Inputs may also be CUDA
torch tensors, in which case results stay on the device.
"""
from __future__ import annotations

import collections
import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import DimensionMismatchError, InvalidFactorError

# ---------------------------------------------------------------------------
# device plumbing (torch owns device memory; libnpcg owns pattern analyses)
# ---------------------------------------------------------------------------


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise _native.NativeUnavailableError("CUDA is not available; libnpcg has no CPU fallback")
    return torch


def to_device(x, dtype=None):
    """numpy / torch -> contiguous CUDA float64 tensor (no copy if already there)."""
    torch = _torch()
    if isinstance(x, torch.Tensor):
        t = x
        if not t.is_cuda:
            t = t.cuda(non_blocking=True)
    else:
        t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()
    return t.to(dtype or torch.float64).contiguous()


_VALIDATED: dict = {}  # (id(row_ptr), id(col_idx), n) -> (row_ptr, col_idx) that passed the index checks

# Pinned host buffers for results handed back as numpy arrays: a device -> pageable copy of a
# fresh 33 MB array runs at ~2 GB/s (page faults + staging; 14.7 ms for config 2's solutions),
# a copy into pinned memory at the link rate (1.3 ms). A buffer is reused once the array that
# was handed out on it (and every view of it) is gone.
_HOST_POOL: list = []  # [pinned tensor, weakref to the array last handed out | None]
_HOST_POOL_MAX = 6


def to_host(t):
    """CUDA tensor -> numpy array (same shape) backed by pooled pinned memory."""
    import weakref
    torch = _torch()
    t = t.contiguous()
    n, slot = t.numel(), None
    for entry in _HOST_POOL:
        buf, ref = entry
        if buf.dtype == t.dtype and buf.numel() >= n and (ref is None or ref() is None):
            if slot is None or buf.numel() < slot[0].numel():
                slot = entry
    if slot is None:
        if len(_HOST_POOL) >= _HOST_POOL_MAX:  # drop a free buffer (or fall back to a pageable copy)
            free = [e for e in _HOST_POOL if e[1] is None or e[1]() is None]
            if not free:
                return t.cpu().numpy()
            _HOST_POOL.remove(min(free, key=lambda e: e[0].numel()))
        slot = [torch.empty(max(n, 1), dtype=t.dtype, pin_memory=True), None]
        _HOST_POOL.append(slot)
    view = slot[0][:n].view(t.shape)
    view.copy_(t)
    arr = view.numpy()
    slot[1] = weakref.ref(arr)
    return arr


def is_device(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor) and x.is_cuda


class DevicePattern:
    """Handle on one analysed sparsity pattern (npcg_pattern)."""

    def __init__(self, n, row_ptr, col_idx, factor=False):
        lib = _native.lib()
        h = ctypes.c_void_p()
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(col_idx, dtype=np.int64)
        rc = lib.npcg_pattern_create(n, rp.ctypes.data, ci.ctypes.data if len(ci) else None,
                                     _native.PATTERN_FACTOR if factor else 0, ctypes.byref(h))
        _native.check(rc)
        self.handle = h
        self.n = int(n)
        self.nnz = int(rp[-1]) if len(rp) else 0
        self._solvers = {}
        self._lib = lib

    def info(self) -> _native.PatternInfo:
        out = _native.PatternInfo()
        _native.check(self._lib.npcg_pattern_get_info(self.handle, ctypes.byref(out)))
        return out

    @property
    def nnz_lower(self) -> int:
        return int(self.info().nnz_lower)

    def solver(self, factor_pattern, B, tag=0):
        """Cached npcg_solver for (this A pattern, factor pattern or None, B);
        ``tag`` keeps concurrent solves (one per stream) on distinct solvers."""
        key = (id(factor_pattern), B, tag)
        s = self._solvers.get(key)
        if s is None:
            h = ctypes.c_void_p()
            fh = factor_pattern.handle if factor_pattern is not None else None
            _native.check(self._lib.npcg_solver_create(self.handle, fh, B, ctypes.byref(h)))
            s = (h, factor_pattern)  # keep the factor pattern alive with the solver
            self._solvers[key] = s
        return s[0]

    def __del__(self):
        try:
            for h, _ in self._solvers.values():
                self._lib.npcg_solver_destroy(h)
            self._lib.npcg_pattern_destroy(self.handle)
        except Exception:  # interpreter shutdown
            pass


_PATTERNS: "collections.OrderedDict" = collections.OrderedDict()
_PATTERN_CACHE_SIZE = 32


def device_pattern(n, row_ptr, col_idx, factor=False) -> DevicePattern:
    """Pattern handle shared by every matrix built on the same index arrays
    (one analysis per mesh). Keyed on array identity; the cache holds the
    arrays so the identity stays valid. ``factor=True`` additionally requires
    a full diagonal and a symmetric pattern (DataFormatError otherwise, as
    graph_from_system raises, gnn.py:79-82)."""
    key = (id(row_ptr), id(col_idx), int(n))
    hit = _PATTERNS.get(key)
    if hit is not None:
        _PATTERNS.move_to_end(key)
        pat = hit[2]
    else:
        pat = DevicePattern(n, row_ptr, col_idx, False)
        _PATTERNS[key] = (row_ptr, col_idx, pat)
        while len(_PATTERNS) > _PATTERN_CACHE_SIZE:
            _PATTERNS.popitem(last=False)
    if factor:
        info = pat.info()
        if not info.full_diagonal:
            from .errors import DataFormatError
            raise DataFormatError("matrix is missing explicit diagonal entries")
        if not info.structurally_symmetric:
            from .errors import DataFormatError
            raise DataFormatError("matrix values are not symmetric")
    return pat


# ---------------------------------------------------------------------------
# storage (sparse.py:30-166)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class SparseMatrixCsr:
    """Square CSR matrix; invariants as in sparse.py:44-65 (checked here)."""

    n: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "row_ptr", np.ascontiguousarray(self.row_ptr, dtype=np.int64))
        object.__setattr__(self, "col_idx", np.ascontiguousarray(self.col_idx, dtype=np.int64))
        object.__setattr__(self, "values", np.ascontiguousarray(self.values, dtype=np.float64))
        n, rp, ci = self.n, self.row_ptr, self.col_idx
        object.__setattr__(self, "_dev_vals", None)
        object.__setattr__(self, "_sym", None)
        # index arrays already validated (same objects: one mesh, many matrices) are not
        # walked again; like the device pattern, the cache is keyed on array identity and
        # holds the arrays
        key = (id(rp), id(ci), int(n))
        hit = _VALIDATED.get(key)
        if hit is not None and hit[0] is rp and hit[1] is ci:
            if len(ci) != len(self.values):
                raise DimensionMismatchError("row_ptr endpoints disagree with nnz")
            return
        if n < 0 or rp.shape != (n + 1,):
            raise DimensionMismatchError(f"row_ptr must have length n+1={n + 1}")
        if rp[0] != 0 or rp[-1] != len(ci) or len(ci) != len(self.values):
            raise DimensionMismatchError("row_ptr endpoints disagree with nnz")
        if np.any(np.diff(rp) < 0):
            raise DimensionMismatchError("row_ptr must be non-decreasing")
        if len(ci) and (ci.min() < 0 or ci.max() >= n):
            raise DimensionMismatchError("column index out of range")
        if len(ci) > 1:
            ok = np.diff(ci) > 0
            heads = rp[1:-1]
            heads = heads[(heads > 0) & (heads < len(ci))]
            ok[heads - 1] = True  # pairs straddling a row boundary are exempt
            if not np.all(ok):
                raise DimensionMismatchError("columns must strictly increase within rows")
        _VALIDATED[key] = (rp, ci)
        while len(_VALIDATED) > 64:
            _VALIDATED.pop(next(iter(_VALIDATED)))

    # -- constructors (sparse.py:69-108) --------------------------------------

    @staticmethod
    def from_coo(n, rows, cols, vals):
        """Triplets -> CSR; duplicates summed in ascending input order."""
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        vals = np.asarray(vals, dtype=np.float64)
        if not (len(rows) == len(cols) == len(vals)):
            raise DimensionMismatchError("COO arrays must share a length")
        if len(rows) == 0:
            return SparseMatrixCsr(n, np.zeros(n + 1, dtype=np.int64), rows, vals)
        order = np.lexsort((cols, rows))
        r, c, v = rows[order], cols[order], vals[order]
        head = np.ones(len(r), dtype=bool)
        head[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
        starts = np.flatnonzero(head)
        summed = np.add.reduceat(v, starts)
        rp = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(np.bincount(r[starts], minlength=n), out=rp[1:])
        return SparseMatrixCsr(n, rp, c[starts], summed)

    @staticmethod
    def from_dense(dense):
        dense = np.asarray(dense, dtype=np.float64)
        if dense.ndim != 2 or dense.shape[0] != dense.shape[1]:
            raise DimensionMismatchError("dense input must be square")
        rows, cols = np.nonzero(dense)
        return SparseMatrixCsr.from_coo(dense.shape[0], rows, cols, dense[rows, cols])

    @staticmethod
    def identity(n):
        idx = np.arange(n, dtype=np.int64)
        return SparseMatrixCsr(n, np.arange(n + 1, dtype=np.int64), idx, np.ones(n))

    # -- views -------------------------------------------------------------------

    @property
    def nnz(self):
        return len(self.values)

    def row_indices(self):
        return np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.row_ptr))

    def to_dense(self):
        out = np.zeros((self.n, self.n))
        out[self.row_indices(), self.col_idx] = self.values
        return out

    def diagonal(self):
        d = np.zeros(self.n)
        rows = self.row_indices()
        on = rows == self.col_idx
        d[rows[on]] = self.values[on]
        return d

    def has_full_diagonal(self):
        return np.count_nonzero(self.row_indices() == self.col_idx) == self.n

    def is_symmetric(self):
        """Exact value symmetry (sparse.py:137-147, np.array_equal semantics),
        checked on the device (once: the values are immutable, like the
        device copy they are checked on)."""
        if self._sym is None:
            pat = self.device_pattern()
            ok = (ctypes.c_int32 * 1)()
            if pat_symmetric(pat):
                vals = self.device_values()
                _native.check(_native.lib().npcg_check_symmetric_values(pat.handle, 1, _native.ptr(vals), 0,
                                                                        ok, _native.stream_handle()))
            object.__setattr__(self, "_sym", bool(ok[0]))
        return self._sym

    def strict_lower(self):
        rows = self.row_indices()
        keep = rows > self.col_idx
        return SparseMatrixCsr.from_coo(self.n, rows[keep], self.col_idx[keep], self.values[keep])

    def submatrix(self, keep):
        keep = np.asarray(keep, dtype=np.int64)
        remap = -np.ones(self.n, dtype=np.int64)
        remap[keep] = np.arange(len(keep), dtype=np.int64)
        rows = remap[self.row_indices()]
        cols = remap[self.col_idx]
        sel = (rows >= 0) & (cols >= 0)
        return SparseMatrixCsr.from_coo(len(keep), rows[sel], cols[sel], self.values[sel])

    def scaled(self, factor):
        return SparseMatrixCsr(self.n, self.row_ptr, self.col_idx, self.values * factor)

    def with_values(self, values):
        """Same pattern (and device analysis), new values."""
        return SparseMatrixCsr(self.n, self.row_ptr, self.col_idx, values)

    # -- device views --------------------------------------------------------------

    def device_pattern(self, factor=False) -> DevicePattern:
        return device_pattern(self.n, self.row_ptr, self.col_idx, factor)

    def device_values(self):
        """Values on the device (uploaded once; matrices are immutable)."""
        if self._dev_vals is None:
            object.__setattr__(self, "_dev_vals", to_device(self.values))
        return self._dev_vals


def pat_symmetric(pat: DevicePattern) -> bool:
    return bool(pat.info().structurally_symmetric)


# ---------------------------------------------------------------------------
# LDL^T factor (sparse.py:169-204)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class LowerFactor:
    """Unit-lower LDL^T factor P = (I + L) D (I + L)^T, L strictly lower."""

    n: int
    strict_lower: SparseMatrixCsr
    diag: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "diag", np.ascontiguousarray(self.diag, dtype=np.float64))
        if self.strict_lower.n != self.n or self.diag.shape != (self.n,):
            raise DimensionMismatchError("factor parts disagree on dimension")
        sl = self.strict_lower
        if sl.nnz and not np.all(sl.row_indices() > sl.col_idx):
            raise InvalidFactorError("strict_lower must only hold entries below the diagonal")
        if not np.all(np.isfinite(self.diag)) or np.any(self.diag <= 0):
            raise InvalidFactorError("diagonal must be finite and strictly positive")
        if sl.nnz and not np.all(np.isfinite(sl.values)):
            raise InvalidFactorError("factor values must be finite")
        object.__setattr__(self, "_dev", None)

    @property
    def nnz_lower(self):
        return self.strict_lower.nnz

    def unit_lower_dense(self):
        return np.eye(self.n) + self.strict_lower.to_dense()

    def to_dense(self):
        b = self.unit_lower_dense()
        return (b * self.diag) @ b.T

    def device(self):
        """(pattern, S, D) on the device. The solve pattern is the symmetric
        closure L + L^T + I; S holds L' on both triangles (npcg.h)."""
        if self._dev is None:
            sl = self.strict_lower
            rows = sl.row_indices()
            n = self.n
            ar = np.arange(n, dtype=np.int64)
            rr = np.concatenate([rows, sl.col_idx, ar])
            cc = np.concatenate([sl.col_idx, rows, ar])
            sym = SparseMatrixCsr.from_coo(n, rr, cc, np.zeros(len(rr)))
            pat = DevicePattern(n, sym.row_ptr, sym.col_idx, factor=True)
            torch = _torch()
            S = torch.empty(max(sym.nnz, 1), dtype=torch.float64, device="cuda")
            lower = to_device(sl.values) if sl.nnz else S[:1]
            _native.check(_native.lib().npcg_factor_from_lower(pat.handle, 1, _native.ptr(lower), 0,
                                                               _native.ptr(S), _native.stream_handle()))
            object.__setattr__(self, "_dev", (pat, S, to_device(self.diag), sym))
        return self._dev[:3]


# ---------------------------------------------------------------------------
# operations (sparse.py:255-292)
# ---------------------------------------------------------------------------


def spmv_device(A: SparseMatrixCsr, x, B=1, vals=None, vals_batched=False):
    """y = A x on device tensors; x is (n,) or (n, B)."""
    torch = _torch()
    pat = A.device_pattern()
    vals = A.device_values() if vals is None else vals
    y = torch.empty_like(x)
    _native.check(_native.lib().npcg_spmv(pat.handle, B, _native.ptr(vals), int(vals_batched),
                                          _native.ptr(x), _native.ptr(y), _native.stream_handle()))
    return y


def spmv(A: SparseMatrixCsr, x):
    """y = A x (sparse.py:255-262); numpy in -> numpy out, CUDA in -> CUDA out."""
    on_dev = is_device(x)
    shape = tuple(x.shape)
    if shape != (A.n,):
        raise DimensionMismatchError(f"x has shape {shape}, expected ({A.n},)")
    y = spmv_device(A, to_device(x))
    return y if on_dev else y.cpu().numpy()


def ldlt_apply_inverse(F: LowerFactor, r):
    """Solve (I+L) D (I+L)^T z = r (sparse.py:265-275) with the device SpTRSV."""
    on_dev = is_device(r)
    if tuple(r.shape) != (F.n,):
        raise DimensionMismatchError(f"rhs has shape {tuple(r.shape)}, expected ({F.n},)")
    pat, S, D = F.device()
    z = apply_inverse_device(pat, S, False, D, False, to_device(r), 1)
    return z if on_dev else z.cpu().numpy()


def apply_inverse_device(pat, S, s_batched, D, d_batched, r, B):
    torch = _torch()
    z = torch.empty_like(r)
    if pat.n == 0:
        return z
    _native.check(_native.lib().npcg_ldlt_apply_inverse(
        pat.handle, B, _native.ptr(S), int(s_batched), _native.ptr(D), int(d_batched),
        _native.ptr(r), _native.ptr(z), _native.stream_handle()))
    return z


def ldlt_apply(F: LowerFactor, x):
    """y = (I+L) D (I+L)^T x (sparse.py:278-292), as three device products."""
    torch = _torch()
    on_dev = is_device(x)
    if tuple(x.shape) != (F.n,):
        raise DimensionMismatchError(f"x has shape {tuple(x.shape)}, expected ({F.n},)")
    sl = F.strict_lower
    xd = to_device(x)
    if sl.nnz:
        Lt = SparseMatrixCsr.from_coo(F.n, sl.col_idx, sl.row_indices(), sl.values)
        t = xd + spmv_device(Lt, xd)
    else:
        t = xd.clone()
    t = t * to_device(F.diag)
    y = t + spmv_device(sl, t) if sl.nnz else t
    _ = torch
    return y if on_dev else y.cpu().numpy()
