"""CPU restatement ("port") of the reference NeuralPCG solve path.

TEST INFRASTRUCTURE ONLY -- this module is the parity checker. It may be
imported by ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py``; the product package
(``paper_2305_16432_b200``) never imports it and has no CPU fallback.

It restates, as plain functions over numpy arrays (no autodiff tape), the
reference package ``pcgkit`` (read-only at /root/reference, not available on
the GPU box):

* CSR helpers              -- pkg/src/pcgkit/sparse.py:30-166
* spmv / ldlt_apply_inverse -- sparse.py:213-275 (loops in oracle/kernels.c)
* graph construction       -- gnn.py:42-98
* model parameters / init  -- gnn.py:106-184, checkpoints gnn.py:335-374
* GNN forward (inference)  -- gnn.py:218-270 over autodiff.py:113-253
* symmetrize + assemble    -- gnn.py:278-318
* PCG                      -- pcg.py:75-176

Pinning: tests/test_oracle_golden.py checks this port bitwise against
golden vectors produced by running the reference itself
(tests/golden/make_golden.py); so "parity pinned".
"""
from __future__ import annotations

import ctypes
import json
import os
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None


def build():
    """Compile oracle/kernels.c (gcc) into oracle/_build/liboracle.so."""
    import subprocess
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def _kernels():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        lib = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        I = ctypes.c_int64
        lib.oracle_spmv.argtypes = [I, P, P, P, P, P]
        lib.oracle_forward_unit.argtypes = [I, P, P, P, P, P]
        lib.oracle_backward_unit_t.argtypes = [I, P, P, P, P]
        lib.oracle_ldlt_apply_inverse.argtypes = [I, P, P, P, P, P, P]
        lib.oracle_segment_sum_sorted.argtypes = [I, I, P, P, P]
        _lib = lib
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------------------
# CSR (sparse.py:30-166). A matrix is a tuple-like Csr(n, row_ptr, col, val).
# ---------------------------------------------------------------------------


class Csr:
    __slots__ = ("n", "row_ptr", "col_idx", "values")

    def __init__(self, n, row_ptr, col_idx, values):
        self.n = int(n)
        self.row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
        self.col_idx = np.ascontiguousarray(col_idx, dtype=np.int64)
        self.values = np.ascontiguousarray(values, dtype=np.float64)

    @property
    def nnz(self):
        return len(self.values)

    def rows(self):
        return np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.row_ptr))

    def dense(self):
        out = np.zeros((self.n, self.n))
        out[self.rows(), self.col_idx] = self.values
        return out


def csr_from_coo(n, rows, cols, vals):
    """Triplets -> CSR; duplicates summed in input order (sparse.py:69-94)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    if len(rows) == 0:
        return Csr(n, np.zeros(n + 1, dtype=np.int64), rows, vals)
    order = np.lexsort((cols, rows))
    r, c, v = rows[order], cols[order], vals[order]
    head = np.ones(len(r), dtype=bool)
    head[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
    starts = np.flatnonzero(head)
    total = np.add.reduceat(v, starts)
    counts = np.bincount(r[starts], minlength=n)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    return Csr(n, row_ptr, c[starts], total)


def diagonal(A):
    d = np.zeros(A.n)
    r = A.rows()
    on = r == A.col_idx
    d[r[on]] = A.values[on]
    return d


def strict_lower(A):
    r = A.rows()
    keep = r > A.col_idx
    return csr_from_coo(A.n, r[keep], A.col_idx[keep], A.values[keep])


def is_symmetric(A):
    r = A.rows()
    a = np.lexsort((A.col_idx, r))
    b = np.lexsort((r, A.col_idx))
    return (np.array_equal(r[a], A.col_idx[b]) and np.array_equal(A.col_idx[a], r[b])
            and np.array_equal(A.values[a], A.values[b]))


def spmv(A, x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(A.n)
    _kernels().oracle_spmv(A.n, _p(A.row_ptr), _p(A.col_idx), _p(A.values), _p(x), _p(y))
    return y


class Factor:
    """Unit-lower LDL^T factor (sparse.py:169-204): P = (I+L) D (I+L)^T."""

    __slots__ = ("n", "lower", "diag")

    def __init__(self, n, lower, diag):
        self.n, self.lower = n, lower
        self.diag = np.ascontiguousarray(diag, dtype=np.float64)

    def apply_inverse(self, r):
        r = np.ascontiguousarray(r, dtype=np.float64)
        z = np.empty(self.n)
        L = self.lower
        _kernels().oracle_ldlt_apply_inverse(self.n, _p(L.row_ptr), _p(L.col_idx),
                                             _p(L.values), _p(self.diag), _p(r), _p(z))
        return z

    def dense(self):
        B = np.eye(self.n) + self.lower.dense()
        return (B * self.diag) @ B.T


# ---------------------------------------------------------------------------
# graph (gnn.py:42-98)
# ---------------------------------------------------------------------------


def sorted_stats(values):
    m = len(values)
    if m == 0:
        return 0.0, 1.0
    mean = float(np.sum(np.sort(values)) / m)
    var = float(np.sum(np.sort((values - mean) ** 2)) / m)
    sd = var ** 0.5
    return mean, (sd if sd > 0.0 else 1.0)


class Graph:
    __slots__ = ("n", "src", "dst", "pair", "node_in", "edge_in", "node_stats", "edge_stats")


def graph_from_system(A, b):
    b = np.asarray(b, dtype=np.float64)
    g = Graph()
    g.n = A.n
    g.src = A.rows()
    g.dst = A.col_idx.copy()
    order = np.lexsort((g.src, g.dst))
    g.pair = np.empty(len(order), dtype=np.int64)
    g.pair[order] = np.arange(len(order), dtype=np.int64)
    g.node_in = b[:, None].copy()
    g.edge_in = A.values[:, None].copy()
    g.node_stats = sorted_stats(b)
    g.edge_stats = sorted_stats(A.values)
    return g


# ---------------------------------------------------------------------------
# model (gnn.py:106-184, 335-374)
# ---------------------------------------------------------------------------


class Hyper:
    """mode "reference": pcgkit's network (gnn.py:106-147). mode
    "north_star": BASELINE.json's extensions -- node inputs (b_i, boundary
    flag), edge inputs (A_ij, d_1..d_dim, |d|) with d = x_dst - x_src,
    LayerNorm after every encoder / processor MLP, and a factor L with an
    exponentiated diagonal, P = L L^T (no reference code pins these: this
    restatement is their only oracle -- "parity unpinned")."""

    def __init__(self, l=1, h=16, n_mp=5, l_mp=1, h_mp=16, with_x0_head=False,
                 normalize=True, width=16, mode="reference", dim=2):
        self.l, self.h, self.n_mp, self.l_mp, self.h_mp = l, h, n_mp, l_mp, h_mp
        self.with_x0_head, self.normalize, self.width = with_x0_head, normalize, width
        self.mode, self.dim = mode, dim

    @property
    def north_star(self):
        return self.mode == "north_star"


LN_EPS = 1e-5


def layer_specs(hp):
    """(name, fan_in, fan_out) in the reference's draw order (gnn.py:130-147)."""
    out = []

    def stack(prefix, fin, hidden, layers, fout):
        dims = [fin] + [hidden] * layers + [fout]
        for k in range(len(dims) - 1):
            out.append((f"{prefix}.{k}", dims[k], dims[k + 1]))

    F = hp.width
    ns = getattr(hp, "north_star", False)
    stack("node_enc", 2 if ns else 1, hp.h, hp.l, F)
    stack("edge_enc", 2 + hp.dim if ns else 1, hp.h, hp.l, F)
    for r in range(hp.n_mp):
        stack(f"mp{r}.node", 2 * F, hp.h_mp, hp.l_mp, F)
        stack(f"mp{r}.edge", 3 * F, hp.h_mp, hp.l_mp, F)
    stack("edge_dec", F, hp.h, hp.l, 1)
    if hp.with_x0_head:
        stack("node_dec", F, hp.h, hp.l, 1)
    return out


def create_params(hp, seed=0):
    rng = np.random.default_rng(seed)
    last = str(hp.l_mp)
    params = {}
    for name, fi, fo in layer_specs(hp):
        s = (2.0 / (fi + fo)) ** 0.5
        if name.startswith("mp") and name.split(".")[-1] == last:
            s *= 0.1
        params[name + ".w"] = rng.standard_normal((fi, fo)) * s
        params[name + ".b"] = np.zeros(fo)
    for stack_name in ln_stacks(hp):  # LayerNorm gain / shift, no RNG draws
        params[stack_name + ".ln.g"] = np.ones(hp.width)
        params[stack_name + ".ln.b"] = np.zeros(hp.width)
    return params


def ln_stacks(hp):
    """Stacks followed by a LayerNorm (north_star mode): encoders and processors."""
    if not getattr(hp, "north_star", False):
        return []
    out = ["node_enc", "edge_enc"]
    for r in range(hp.n_mp):
        out += [f"mp{r}.node", f"mp{r}.edge"]
    return out


def load_checkpoint(path):
    """Reference checkpoint JSON (gnn.py:356-374); F inferred from shapes."""
    with open(path, encoding="ascii") as fh:
        doc = json.load(fh)
    assert doc["format_version"] == 1
    h = doc["hyper"]
    params = {k: np.array(v["data"], dtype=np.float64).reshape(v["shape"])
              for k, v in doc["tensors"].items()}
    width = params["node_enc.%d.w" % h["l"]].shape[1]
    return Hyper(width=width, **h), params


# ---------------------------------------------------------------------------
# forward (gnn.py:218-270; primitives autodiff.py:113-253)
# ---------------------------------------------------------------------------


def _affine(x, W, b):
    if W.shape[1] == 1:  # column-by-column accumulation (autodiff.py:127-131)
        out = np.tile(b, (x.shape[0], 1))
        for f in range(x.shape[1]):
            out += x[:, f, None] * W[f, None, :]
        return out
    return x @ W + b


def _mlp(params, prefix, x, layers):
    for k in range(layers + 1):
        x = _affine(x, params[f"{prefix}.{k}.w"], params[f"{prefix}.{k}.b"])
        if k < layers:
            x = np.where(x > 0.0, x, 0.0)
    return x


def _segment_sum(x, seg, n):
    """Canonical-order segment sum (autodiff.py:221-243). CSR-ordered
    segments (non-decreasing seg, the GNN's case) go through the C loop in
    kernels.c, which sorts each segment's addends in the same lexicographic
    order and sums them like np.add.reduceat; anything else takes the
    lexsort restatement below."""
    out = np.zeros((n, x.shape[1]))
    if x.shape[0] and x.shape[1] and np.all(seg[1:] >= seg[:-1]):
        xc = np.ascontiguousarray(x, dtype=np.float64)
        sc = np.ascontiguousarray(seg, dtype=np.int64)
        _kernels().oracle_segment_sum_sorted(x.shape[0], x.shape[1], _p(xc), _p(sc), _p(out))
        return out
    return _segment_sum_lexsort(x, seg, n)


def _segment_sum_lexsort(x, seg, n):
    out = np.zeros((n, x.shape[1]))
    if x.shape[0]:
        keys = tuple(x[:, c] for c in range(x.shape[1] - 1, -1, -1)) + (seg,)
        order = np.lexsort(keys)
        sv, ss = x[order], seg[order]
        starts = np.r_[0, np.flatnonzero(np.diff(ss)) + 1]
        out[ss[starts]] = np.add.reduceat(sv, starts, axis=0)
    return out


def _layer_norm(params, prefix, x):
    """LayerNorm over the feature axis (population variance, eps LN_EPS),
    then gain and shift: the north_star MLPs' output normalisation."""
    mu = x.mean(axis=1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=1, keepdims=True)
    return (x - mu) / np.sqrt(var + LN_EPS) * params[prefix + ".ln.g"] + params[prefix + ".ln.b"]


def _mlp_ln(params, prefix, x, layers, ln):
    y = _mlp(params, prefix, x, layers)
    return _layer_norm(params, prefix, y) if ln else y


def north_star_inputs(g, b, A, pos, boundary):
    """Node inputs (b_i, boundary flag) and edge inputs (A_ij, d, |d|) with
    d = pos[dst] - pos[src], every column standardised per graph with the
    reference's sorted statistics (gnn.py:42-51)."""
    b = np.asarray(b, dtype=np.float64)
    pos = np.asarray(pos, dtype=np.float64)
    flag = np.asarray(boundary, dtype=np.float64)
    node = np.stack([b, flag], axis=1)
    d = pos[g.dst] - pos[g.src]
    dist = np.sqrt(np.sum(d * d, axis=1))
    edge = np.concatenate([A.values[:, None], d, dist[:, None]], axis=1)

    def standardise(x):
        cols = []
        for c in range(x.shape[1]):
            mu, sd = sorted_stats(x[:, c])
            cols.append((x[:, c] - mu) / sd)
        return np.stack(cols, axis=1)

    return standardise(node), standardise(edge)


def gnn_run(hp, params, g):
    """Returns (edge scalars M[m], node scalars x0[n] or None). In north_star
    mode g carries the standardised mesh inputs (north_star_inputs)."""
    ln = getattr(hp, "north_star", False)
    node_in, edge_in = g.node_in, g.edge_in
    if not ln and hp.normalize:
        node_in = (node_in - g.node_stats[0]) / g.node_stats[1]
        edge_in = (edge_in - g.edge_stats[0]) / g.edge_stats[1]
    v = _mlp_ln(params, "node_enc", node_in, hp.l, ln)
    e = _mlp_ln(params, "edge_enc", edge_in, hp.l, ln)
    for r in range(hp.n_mp):
        agg = _segment_sum(e * v[g.dst], g.src, g.n)
        v = _mlp_ln(params, f"mp{r}.node", np.concatenate((v, agg), axis=1), hp.l_mp, ln)
        e = _mlp_ln(params, f"mp{r}.edge",
                    np.concatenate((e, v[g.src], v[g.dst]), axis=1), hp.l_mp, ln)
    M = _mlp(params, "edge_dec", e, hp.l).reshape(-1)
    x0 = _mlp(params, "node_dec", v, hp.l).reshape(-1) if hp.with_x0_head else None
    return M, x0


def symmetrize(M, g):
    idx = np.flatnonzero(g.src > g.dst)
    return 0.5 * (M[idx] + M[g.pair[idx]])


def assemble(lower_values, A):
    d = diagonal(A)
    if np.any(d <= 0.0):
        raise ValueError("nonpositive diagonal at row %d" % int(np.argmax(d <= 0.0)))
    pat = strict_lower(A)
    return Factor(A.n, Csr(A.n, pat.row_ptr, pat.col_idx, lower_values), d.copy())


def assemble_exp(M, g, A):
    """north_star factor P = L L^T: L_ii = exp(M_ii) (the self-loop outputs),
    L_ij = (M_ij + M_ji) / 2 below the diagonal. Returned in the unit-lower
    LDL^T form the solver applies, U = L diag(L)^-1 and D = diag(L)^2, so
    P = U D U^T exactly in real arithmetic."""
    lower = symmetrize(M, g)
    diag_slots = np.flatnonzero(g.src == g.dst)
    d = np.exp(M[diag_slots])  # one per row, in row order (CSR)
    pat = strict_lower(A)
    rows = pat.rows()
    U = lower / d[pat.col_idx]
    if not (np.all(np.isfinite(U)) and np.all(np.isfinite(d)) and np.all(d > 0.0)):
        raise ValueError("factor values must be finite with a positive diagonal")
    return Factor(A.n, Csr(A.n, pat.row_ptr, pat.col_idx, U), d * d)


def build_learned(hp, params, A, b, mesh=None):
    g = graph_from_system(A, b)
    if getattr(hp, "north_star", False):
        g.node_in, g.edge_in = north_star_inputs(g, b, A, *mesh)
        M, _ = gnn_run(hp, params, g)
        return assemble_exp(M, g, A)
    M, _ = gnn_run(hp, params, g)
    return assemble(symmetrize(M, g), A)


# ---------------------------------------------------------------------------
# PCG (pcg.py:75-176)
# ---------------------------------------------------------------------------


class Report:
    __slots__ = ("thresholds", "iterations_to", "seconds_to", "final_relative_residual",
                 "converged", "history", "iterations", "breakdown")


def pcg_solve(A, b, P=None, thresholds=(1e-2, 1e-4, 1e-6, 1e-8, 1e-10, 1e-12),
              max_iter=None, x0=None, absolute=False):
    """Faithful restatement; breakdown is reported (rep.breakdown=k) instead
    of raised so batch drivers can keep going."""
    thresholds = tuple(float(t) for t in thresholds)
    b = np.asarray(b, dtype=np.float64)
    max_iter = max_iter if max_iter is not None else 10 * A.n
    t_min = thresholds[-1]
    start = time.perf_counter()
    it_to, sec_to = {}, {}
    rep = Report()
    rep.thresholds, rep.iterations_to, rep.seconds_to, rep.breakdown = thresholds, it_to, sec_to, None
    apply = (lambda r: r.copy()) if P is None else P.apply_inverse

    def finish(x, rel, conv, hist, k):
        rep.final_relative_residual, rep.converged, rep.history, rep.iterations = rel, conv, hist, k
        return x, rep

    norm_b = float(np.linalg.norm(b))
    if norm_b == 0.0:
        for t in thresholds:
            it_to[t] = 0
            sec_to[t] = time.perf_counter() - start
        return finish(np.zeros(A.n), 0.0, True, [0.0], 0)
    scale = 1.0 if absolute else norm_b
    if x0 is not None:
        x = np.array(x0, dtype=np.float64)
        r = b - spmv(A, x)
    else:
        x = np.zeros(A.n)
        r = b.copy()
    hist = [float(np.linalg.norm(r))]
    rel = hist[0] / scale

    def record(k, v):
        for t in thresholds:
            if t not in it_to and v <= t:
                it_to[t] = k
                sec_to[t] = time.perf_counter() - start

    record(0, rel)
    if rel <= t_min:
        return finish(x, rel, True, hist, 0)
    z = apply(r)
    p = z.copy()
    rz = float(r @ z)
    conv = False
    k = 0
    while k < max_iter:
        k += 1
        Ap = spmv(A, p)
        pAp = float(p @ Ap)
        if pAp <= 0.0:
            rep.breakdown = k
            return finish(x, rel, False, hist, k)
        alpha = rz / pAp
        x += alpha * p
        r -= alpha * Ap
        rn = float(np.linalg.norm(r))
        hist.append(rn)
        rel = rn / scale
        if rel <= t_min:
            rt = b - spmv(A, x)
            rel_t = float(np.linalg.norm(rt)) / scale
            if rel_t <= t_min:
                record(k, max(rel, rel_t))
                rel = rel_t
                conv = True
                break
            record(k, rel_t)
            r = rt
            hist[-1] = float(np.linalg.norm(r))
            rel = rel_t
            z = apply(r)
            p = z.copy()
            rz = float(r @ z)
            continue
        record(k, rel)
        z = apply(r)
        rz_new = float(r @ z)
        beta = rz_new / rz
        p = z + beta * p
        rz = rz_new
    if not conv:
        rel = float(np.linalg.norm(b - spmv(A, x))) / scale
    return finish(x, rel, conv, hist, k)
