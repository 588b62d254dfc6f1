"""Preconditioned conjugate gradients on the device (mirrors pcgkit.pcg,
/root/reference/pkg/src/pcgkit/pcg.py:1-176).

``pcg_solve`` keeps the reference signature and semantics -- relative
residual on the recurrence, multi-threshold crossing record, from-scratch
residual check at the first crossing with restart on drift, max_iter =
10 n default, zero right-hand side -> 0 iterations, BreakdownError when
p'Ap <= 0, history of length iterations + 1. The whole loop runs in
libnpcg (npcg_pcg_solve): per-system alpha / beta / thresholds / status
live on the device and the host only polls an "active systems" counter
every few passes. ``pcg_solve_batch`` solves B right-hand sides (or B
systems sharing one pattern) in one loop.
"""
from __future__ import annotations

import ctypes
import os
import threading
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import BreakdownError, DimensionMismatchError
from .sparse import SparseMatrixCsr, is_device, spmv_device, to_device, to_host, _torch

DEFAULT_THRESHOLDS = (1e-2, 1e-4, 1e-6, 1e-8, 1e-10, 1e-12)


@dataclass(frozen=True)
class SolveOptions:
    thresholds: tuple = DEFAULT_THRESHOLDS
    max_iter: int | None = None  # defaults to 10*n at solve time
    x0: object = None
    absolute: bool = False

    def __post_init__(self):
        ts = tuple(float(t) for t in self.thresholds)
        object.__setattr__(self, "thresholds", ts)
        if not ts:
            raise DimensionMismatchError("at least one threshold required")
        if len(ts) > _native.MAX_THRESHOLDS:
            raise DimensionMismatchError(f"at most {_native.MAX_THRESHOLDS} thresholds")
        if any(not (0.0 < t < 1.0) for t in ts):
            raise DimensionMismatchError("thresholds must lie in (0, 1)")
        if any(a <= b for a, b in zip(ts, ts[1:])):
            raise DimensionMismatchError("thresholds must be strictly decreasing")
        if self.max_iter is not None and self.max_iter < 1:
            raise DimensionMismatchError("max_iter must be at least 1")


@dataclass
class SolveReport:
    thresholds: tuple
    iterations_to: dict
    seconds_to: dict
    final_relative_residual: float
    converged: bool
    history: list = field(default_factory=list)
    iterations: int = 0
    status: int = _native.STATUS_CONVERGED

    def at(self, threshold: float):
        if threshold in self.iterations_to:
            return self.iterations_to[threshold], self.seconds_to[threshold]
        return None


class _Identity:
    kind = "identity"

    @staticmethod
    def apply_inverse(r):
        return r.copy() if not is_device(r) else r.clone()


IDENTITY_PRECONDITIONER = _Identity()


def _device_factor(P):
    if P is None or P is IDENTITY_PRECONDITIONER:
        return None
    if hasattr(P, "device_factor"):
        return P.device_factor()
    return False  # foreign Python preconditioner


def pcg_solve(A: SparseMatrixCsr, b, P=None, opts: SolveOptions | None = None):
    """Solve A x = b; returns (x, SolveReport). numpy b -> numpy x; CUDA b -> CUDA x."""
    opts = opts or SolveOptions()
    on_dev = is_device(b)
    if tuple(b.shape) != (A.n,):
        raise DimensionMismatchError(f"rhs length {tuple(b.shape)} does not match n={A.n}")
    if opts.x0 is not None and tuple(np.shape(opts.x0)) != (A.n,):
        raise DimensionMismatchError("x0 length does not match n")
    fac = _device_factor(P)
    if fac is False:
        x, rep = _pcg_foreign(A, b, P, opts)
    else:
        X, reps = _pcg_device(A, to_device(b).view(A.n, 1), fac, opts, batch=1)
        x, rep = X.view(A.n), reps[0]
    if rep.status == _native.STATUS_BREAKDOWN:
        raise BreakdownError(
            f"p'Ap <= 0 at iteration {rep.iterations}: matrix not SPD or preconditioner invalid")
    return (x if on_dev else to_host(x)), rep


def pcg_solve_batch(A, B_rhs, P=None, opts: SolveOptions | None = None, *, values=None,
                    with_history=True, profile=False):
    """Batched solve: B_rhs is (n, B). A is shared, or ``values`` (nnz, B)
    gives B distinct matrices on A's pattern. P is None or a (batched)
    FactorPreconditioner. Returns (X (n, B), [SolveReport] * B); breakdown is
    reported per system (report.status) instead of raised."""
    opts = opts or SolveOptions()
    on_dev = is_device(B_rhs)
    Bm = to_device(B_rhs)
    if Bm.dim() != 2 or Bm.shape[0] != A.n:
        raise DimensionMismatchError("B_rhs must be (n, B)")
    fac = _device_factor(P)
    if fac is False:
        raise TypeError("pcg_solve_batch needs a device preconditioner (FactorPreconditioner) or None")
    X, reps = _pcg_device(A, Bm, fac, opts, batch=Bm.shape[1], values=values,
                          with_history=with_history, profile=profile)
    return (X if on_dev else to_host(X)), reps


LAST_PROFILE: dict = {}  # filled by a profiled solve: per-kernel-class ms / launches / passes

# A batch can be solved as several independent sub-batches, each on its own
# CUDA stream driven by its own host thread (NPCG_STREAMS=2): one half's
# wavefront solves overlap the other half's SpMV / vector updates. Measured at
# config 2 (64 right-hand sides): a ~1100-iteration solve gains 6 % in the PCG
# call (212 vs 226 ms), a ~105-iteration solve (trained weights) loses 30 %
# (29 vs 22 ms: per-sub-batch setup, two wasted tail chunks, host threads) --
# so one stream is the default.
SPLIT_STREAMS = int(os.environ.get("NPCG_STREAMS", "1"))
SPLIT_MIN_BATCH = 16
_STREAMS: list = []


def _side_streams(k):
    torch = _torch()
    dev = torch.cuda.current_device()
    mine = [st for st in _STREAMS if st.device.index == dev]
    while len(mine) < k:
        mine.append(torch.cuda.Stream(device=dev))
        _STREAMS.append(mine[-1])
    return mine[:k]


def _has_line_schedule(A, fac):
    """Whether the factor pattern's solves take the line wavefront (2-D
    meshes); the others run grid-synchronous level kernels, which use the
    whole GPU per launch and gain nothing from a stream split."""
    if fac is None:
        return True  # identity preconditioner: keep the split
    pat = fac[0]
    lines = ctypes.c_int32()
    _native.check(_native.lib().npcg_pattern_line_info(pat.handle, ctypes.byref(lines), None, None, None, 1))
    return lines.value > 0


def _pcg_device(A, Bm, fac, opts, batch, values=None, with_history=True, profile=False):
    k = SPLIT_STREAMS if batch >= SPLIT_MIN_BATCH and SPLIT_STREAMS > 1 else 1
    if k > 1 and not _has_line_schedule(A, fac):
        k = 1
    if k == 1:
        X, reps, prof = _pcg_device_one(A, Bm, fac, opts, batch, values, with_history, profile)
        LAST_PROFILE.clear()
        LAST_PROFILE.update(prof)
        return X, reps
    torch = _torch()
    n = A.n
    if fac is not None and fac[5] not in (1, batch):
        raise DimensionMismatchError("batched factor does not match the batch")
    cuts = [batch * i // k for i in range(k + 1)]
    caller = torch.cuda.current_stream()
    streams = _side_streams(k)
    results = [None] * k
    errors = [None] * k

    def cols(t, lo, hi, rows):  # columns [lo, hi) of a column-minor (rows, batch) tensor
        return t.view(rows, batch)[:, lo:hi].contiguous()

    dev = torch.cuda.current_device()

    def part(i):
        lo, hi = cuts[i], cuts[i + 1]
        try:
            torch.cuda.set_device(dev)  # a new host thread starts on device 0
            with torch.cuda.stream(streams[i]):
                f = fac
                if fac is not None and fac[5] != 1:  # per-system factors: this part's columns
                    patF, S, sb, D, db, FB = fac
                    Sp = cols(S, lo, hi, patF.nnz).view(-1) if sb else S
                    Dp = cols(D, lo, hi, n).view(-1) if db else D
                    f = (patF, Sp, sb, Dp, db, hi - lo)
                v = None if values is None else to_device(values)[:, lo:hi].contiguous()
                results[i] = _pcg_device_one(A, Bm[:, lo:hi].contiguous(), f, opts, hi - lo, v, with_history,
                                             profile, tag=i + 1)
        except BaseException as e:  # re-raised in the caller
            errors[i] = e

    for st in streams:
        st.wait_stream(caller)
    threads = [threading.Thread(target=part, args=(i,)) for i in range(1, k)]
    for th in threads:
        th.start()
    part(0)
    for th in threads:
        th.join()
    for st in streams:
        caller.wait_stream(st)
    for e in errors:
        if e is not None:
            raise e
    X = torch.cat([r[0] for r in results], dim=1)
    reps = [rep for r in results for rep in r[1]]
    profs = [r[2] for r in results]
    LAST_PROFILE.clear()
    LAST_PROFILE.update(passes=max(p["passes"] for p in profs),
                        iterations=np.concatenate([p["iterations"] for p in profs]),
                        kernel_ms={key: sum(p["kernel_ms"][key] for p in profs) for key in profs[0]["kernel_ms"]},
                        kernel_launches={key: sum(p["kernel_launches"][key] for p in profs)
                                         for key in profs[0]["kernel_launches"]},
                        streams=k)
    return X, reps


def _pcg_device_one(A, Bm, fac, opts, batch, values=None, with_history=True, profile=False, tag=0):
    torch = _torch()
    n, B = A.n, batch
    if B < 1 or B > _native.MAX_BATCH:
        raise DimensionMismatchError(f"batch must be in [1, {_native.MAX_BATCH}]")
    lib = _native.lib()
    patA = A.device_pattern()
    if values is None:
        vals, vb = A.device_values(), 0
    else:
        vals, vb = to_device(values), 1
        if tuple(vals.shape) != (A.nnz, B):
            raise DimensionMismatchError("values must be (nnz, B)")
    if fac is None:
        patF, S, sb, D, db = None, None, 0, None, 0
    else:
        patF, S, sb, D, db, FB = fac
        if patF.n != n:
            raise DimensionMismatchError("factor and matrix disagree on dimension")
        if FB != 1 and FB != B:
            raise DimensionMismatchError("batched factor does not match the batch")
    solver = patA.solver(patF, B, tag)
    max_iter = opts.max_iter if opts.max_iter is not None else 10 * n
    T = len(opts.thresholds)
    o = _native.SolveOpts()
    o.n_thresholds = T
    for i, t in enumerate(opts.thresholds):
        o.thresholds[i] = t
    o.max_iter = max_iter
    o.absolute = int(opts.absolute)
    o.check_every = 0
    o.profile = int(profile)
    o.history = int(with_history)
    kms = np.zeros(_native.PROF_SLOTS, dtype=np.float64)
    kn = np.zeros(_native.PROF_SLOTS, dtype=np.int64)
    x0 = None if opts.x0 is None else to_device(opts.x0).view(n, 1).expand(n, B).contiguous()
    X = torch.empty((n, B), dtype=torch.float64, device="cuda")
    status = np.zeros(B, dtype=np.int32)
    iters = np.zeros(B, dtype=np.int64)
    it_to = np.zeros((B, T), dtype=np.int64)
    sec_to = np.zeros((B, T), dtype=np.float64)
    final = np.zeros(B, dtype=np.float64)
    bd = np.zeros(B, dtype=np.int64)
    rep = _native.SolveReportC()
    rep.status = status.ctypes.data
    rep.iterations = iters.ctypes.data
    rep.iterations_to = it_to.ctypes.data
    rep.seconds_to = sec_to.ctypes.data
    rep.final_relative_residual = final.ctypes.data
    rep.history = None  # fetched below, sized by the iterations actually run
    rep.history_cap = 0
    rep.breakdown_iteration = bd.ctypes.data
    rep.kernel_ms = kms.ctypes.data
    rep.kernel_launches = kn.ctypes.data
    _native.check(lib.npcg_pcg_solve(
        solver, _native.ptr(vals), vb, _native.ptr(S), int(sb), _native.ptr(D), int(db),
        _native.ptr(Bm), _native.ptr(X), _native.ptr(x0), ctypes.byref(o), ctypes.byref(rep),
        _native.stream_handle()))
    if with_history:
        cap = int(iters.max()) + 1 if B else 1
        hist = np.zeros((B, cap), dtype=np.float64)
        _native.check(lib.npcg_solver_history(solver, hist.ctypes.data, cap, cap, _native.stream_handle()))
    prof = dict(passes=int(rep.passes), iterations=iters.copy(),
                kernel_ms={k: float(kms[i]) for i, k in enumerate(_native.PROF_NAMES)},
                kernel_launches={k: int(kn[i]) for i, k in enumerate(_native.PROF_NAMES)})
    reports = []
    for b in range(B):
        k = int(iters[b])
        itd, sd = {}, {}
        for i, t in enumerate(opts.thresholds):
            if it_to[b, i] >= 0:
                itd[t] = int(it_to[b, i])
                sd[t] = float(sec_to[b, i])
        h = hist[b, : k + 1].tolist() if with_history else []
        reports.append(SolveReport(opts.thresholds, itd, sd, float(final[b]),
                                   bool(status[b] == _native.STATUS_CONVERGED), h, k, int(status[b])))
    return X, reports, prof


def _pcg_foreign(A, b, P, opts):
    """pcg.py:75-176 with a user-supplied Python ``apply_inverse`` (numpy in/out):
    SpMV on the device, the preconditioner wherever the caller's code runs."""
    torch = _torch()
    start = time.perf_counter()
    n = A.n
    bd = to_device(b)
    max_iter = opts.max_iter if opts.max_iter is not None else 10 * n
    smallest = opts.thresholds[-1]
    it_to, sec_to = {}, {}

    def record(k, v):
        for t in opts.thresholds:
            if t not in it_to and v <= t:
                it_to[t] = k
                sec_to[t] = time.perf_counter() - start

    def pinv(r):
        z = P.apply_inverse(r.cpu().numpy())
        return to_device(z)

    norm_b = float(torch.linalg.vector_norm(bd))
    if norm_b == 0.0:
        for t in opts.thresholds:
            it_to[t] = 0
            sec_to[t] = time.perf_counter() - start
        return torch.zeros(n, dtype=torch.float64, device="cuda"), SolveReport(
            opts.thresholds, it_to, sec_to, 0.0, True, [0.0], 0)
    scale = 1.0 if opts.absolute else norm_b
    if opts.x0 is not None:
        x = to_device(opts.x0).clone()
        r = bd - spmv_device(A, x)
    else:
        x = torch.zeros(n, dtype=torch.float64, device="cuda")
        r = bd.clone()
    hist = [float(torch.linalg.vector_norm(r))]
    rel = hist[0] / scale
    record(0, rel)
    if rel <= smallest:
        return x, SolveReport(opts.thresholds, it_to, sec_to, rel, True, hist, 0)
    z = pinv(r)
    p = z.clone()
    rz = float(r @ z)
    conv, k, status = False, 0, _native.STATUS_MAXITER
    while k < max_iter:
        k += 1
        Ap = spmv_device(A, p)
        pAp = float(p @ Ap)
        if pAp <= 0.0:
            return x, SolveReport(opts.thresholds, it_to, sec_to, rel, False, hist, k,
                                  _native.STATUS_BREAKDOWN)
        alpha = rz / pAp
        x += alpha * p
        r -= alpha * Ap
        rn = float(torch.linalg.vector_norm(r))
        hist.append(rn)
        rel = rn / scale
        if rel <= smallest:
            rt = bd - spmv_device(A, x)
            rel_t = float(torch.linalg.vector_norm(rt)) / scale
            if rel_t <= smallest:
                record(k, max(rel, rel_t))
                rel, conv, status = rel_t, True, _native.STATUS_CONVERGED
                break
            record(k, rel_t)
            r = rt
            hist[-1] = float(torch.linalg.vector_norm(r))
            rel = rel_t
            z = pinv(r)
            p = z.clone()
            rz = float(r @ z)
            continue
        record(k, rel)
        z = pinv(r)
        rz_new = float(r @ z)
        p = z + (rz_new / rz) * p
        rz = rz_new
    if not conv:
        rel = float(torch.linalg.vector_norm(bd - spmv_device(A, x))) / scale
    return x, SolveReport(opts.thresholds, it_to, sec_to, rel, conv, hist, k, status)
