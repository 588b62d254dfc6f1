"""Graph-network preconditioner (mirrors pcgkit.gnn,
/root/reference/pkg/src/pcgkit/gnn.py:1-374).

Host side: hyper-parameters, parameter init (same RNG draws as the
reference, so ``create_model(h, seed)`` gives identical weights), reference
checkpoint JSON I/O and the ``GraphData`` view. Device side (libnpcg):
the forward pass, symmetrisation and factor assembly -- ``build_learned``
never leaves the GPU and returns a device-backed ``FactorPreconditioner``
whose factor lives on A's own pattern.

``FEATURE_WIDTH`` is read at call time exactly like the reference
(gnn.py:33, 138), so setting it to 64 selects the latent-64 network.
"""
from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import DataFormatError, DimensionMismatchError, NotSpdError, PcgkitError
from .preconditioners import FactorPreconditioner
from .sparse import LowerFactor, SparseMatrixCsr, is_device, to_device, _torch

FEATURE_WIDTH = 16
CHECKPOINT_VERSION = 1


# ---------------------------------------------------------------------------
# graph view (gnn.py:42-98)
# ---------------------------------------------------------------------------


def _sorted_stats(values) -> tuple[float, float]:
    m = len(values)
    if m == 0:
        return 0.0, 1.0
    mean = float(np.sum(np.sort(values)) / m)
    var = float(np.sum(np.sort((values - mean) ** 2)) / m)
    std = var ** 0.5
    return mean, (std if std > 0.0 else 1.0)


@dataclass(frozen=True)
class GraphData:
    n_nodes: int
    node_features: np.ndarray
    edge_src: np.ndarray
    edge_dst: np.ndarray
    edge_features: np.ndarray
    edge_pair_index: np.ndarray
    node_stats: tuple
    edge_stats: tuple
    matrix: SparseMatrixCsr | None = None  # the system the graph was built from

    @property
    def n_edges(self) -> int:
        return len(self.edge_src)


def graph_from_system(A: SparseMatrixCsr, b) -> GraphData:
    """Host view of the system graph (gnn.py:72-98). build_learned does not
    need it: the device pattern already holds src / pair / lower slots."""
    b = np.asarray(b.cpu().numpy() if is_device(b) else b, dtype=np.float64)
    if b.shape != (A.n,):
        raise DimensionMismatchError(f"b has shape {b.shape}, expected ({A.n},)")
    _check_graph_system(A)
    src = A.row_indices()
    dst = A.col_idx.copy()
    order = np.lexsort((src, dst))
    pair = np.empty(len(order), dtype=np.int64)
    pair[order] = np.arange(len(order), dtype=np.int64)
    return GraphData(A.n, b[:, None].copy(), src, dst, A.values[:, None].copy(), pair,
                     _sorted_stats(b), _sorted_stats(A.values), A)


def _check_graph_system(A: SparseMatrixCsr):
    if not A.has_full_diagonal():
        raise DataFormatError("matrix is missing explicit diagonal entries")
    if not A.is_symmetric():
        raise DataFormatError("matrix values are not symmetric")


# ---------------------------------------------------------------------------
# parameters (gnn.py:106-202)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class GnnHyperParams:
    """gnn.py:106-122, plus ``mode``: "reference" (pcgkit's network) or
    "north_star" -- BASELINE.json's extensions, which no reference code
    pins (the numpy restatement in oracle/port.py is their oracle): node
    inputs (b_i, boundary flag), edge inputs (A_ij, d_1..d_dim, |d|) from the
    mesh, a LayerNorm after every encoder and processor MLP, and the factor
    P = L L^T with L_ii = exp(M_ii) (``dim``: 2 or 3)."""
    l: int = 1
    h: int = 16
    n_mp: int = 5
    l_mp: int = 1
    h_mp: int = 16
    with_x0_head: bool = False
    normalize: bool = True
    mode: str = "reference"
    dim: int = 2

    def __post_init__(self):
        if min(self.l, self.h, self.n_mp, self.l_mp, self.h_mp) < 1:
            raise DimensionMismatchError("all architecture sizes must be >= 1")
        if self.mode not in ("reference", "north_star"):
            raise DimensionMismatchError(f"unknown GNN mode {self.mode!r}")
        if self.dim not in (2, 3):
            raise DimensionMismatchError("dim must be 2 or 3")

    @property
    def north_star(self) -> bool:
        return self.mode == "north_star"


def _mlp_dims(in_dim, hidden, layers, out_dim):
    widths = [in_dim] + [hidden] * layers + [out_dim]
    return list(zip(widths[:-1], widths[1:]))


def _layer_specs(hyper: GnnHyperParams, width: int | None = None) -> list:
    """(name, fan_in, fan_out) in the reference's order (gnn.py:130-147)."""
    specs = []
    f = FEATURE_WIDTH if width is None else width

    def stack(prefix, i, h, l, o):
        for k, (fi, fo) in enumerate(_mlp_dims(i, h, l, o)):
            specs.append((f"{prefix}.{k}", fi, fo))

    stack("node_enc", 2 if hyper.north_star else 1, hyper.h, hyper.l, f)
    stack("edge_enc", 2 + hyper.dim if hyper.north_star else 1, hyper.h, hyper.l, f)
    for r in range(hyper.n_mp):
        stack(f"mp{r}.node", 2 * f, hyper.h_mp, hyper.l_mp, f)
        stack(f"mp{r}.edge", 3 * f, hyper.h_mp, hyper.l_mp, f)
    stack("edge_dec", f, hyper.h, hyper.l, 1)
    if hyper.with_x0_head:
        stack("node_dec", f, hyper.h, hyper.l, 1)
    return specs


def _ln_stacks(hyper: GnnHyperParams) -> list:
    """Stacks followed by a LayerNorm in north_star mode (gain ".ln.g",
    shift ".ln.b", latent width each), in device-blob order."""
    if not hyper.north_star:
        return []
    out = ["node_enc", "edge_enc"]
    for r in range(hyper.n_mp):
        out += [f"mp{r}.node", f"mp{r}.edge"]
    return out


class GnnModel:
    def __init__(self, hyper: GnnHyperParams, params: dict):
        self.hyper = hyper
        self.params = params
        self._dev = None  # (fingerprint, handle)

    def parameter_names(self):
        return sorted(self.params)

    def n_parameters(self):
        return sum(p.size for p in self.params.values())

    def copy(self):
        return GnnModel(self.hyper, {k: v.copy() for k, v in self.params.items()})

    @property
    def width(self) -> int:
        """Latent width implied by the weights (checkpoints do not store it)."""
        return int(self.params[f"node_enc.{self.hyper.l}.w"].shape[1])

    # -- device weights ----------------------------------------------------------------

    def _blob(self):
        parts = []
        for name, fi, fo in _layer_specs(self.hyper, self.width):
            parts.append(np.asarray(self.params[name + ".w"], dtype=np.float64).reshape(-1))
            parts.append(np.asarray(self.params[name + ".b"], dtype=np.float64).reshape(-1))
        for name in _ln_stacks(self.hyper):
            parts.append(np.asarray(self.params[name + ".ln.g"], dtype=np.float64).reshape(-1))
            parts.append(np.asarray(self.params[name + ".ln.b"], dtype=np.float64).reshape(-1))
        return np.ascontiguousarray(np.concatenate(parts))

    def device(self):
        """npcg_gnn handle, rebuilt whenever the parameters change."""
        # cheap fingerprint first (per array: identity, shape, sum and sum of squares -- any
        # in-place edit of the weights changes it); the blob is only formed for an upload
        fp = tuple((k, id(v), v.shape, float(v.sum()), float(np.vdot(v, v))) for k, v in sorted(self.params.items()))
        if self._dev is not None and self._dev[0] == fp:
            return self._dev[1]
        _validate_params(self, self.width)
        blob = self._blob()
        hp = self.hyper
        d = _native.GnnDesc(self.width, hp.h, hp.l, hp.h_mp, hp.l_mp, hp.n_mp, int(hp.normalize),
                            int(hp.with_x0_head), int(hp.north_star), hp.dim)
        lib = _native.lib()
        h = ctypes.c_void_p()
        _native.check(lib.npcg_gnn_create(ctypes.byref(d), blob.ctypes.data, len(blob), ctypes.byref(h)))
        self._release()
        self._dev = (fp, _GnnHandle(lib, h))
        return self._dev[1]

    def _release(self):
        self._dev = None


class _GnnHandle:
    def __init__(self, lib, h):
        self.lib, self.h = lib, h

    def __del__(self):
        try:
            self.lib.npcg_gnn_destroy(self.h)
        except Exception:
            pass


def create_model(hyper: GnnHyperParams = GnnHyperParams(), seed: int = 0) -> GnnModel:
    """Glorot-normal weights (x0.1 on processor output layers), zero biases;
    identical draws to gnn.py:165-184."""
    rng = np.random.default_rng(seed)
    last_mp = str(hyper.l_mp)
    params = {}
    for name, fi, fo in _layer_specs(hyper):
        scale = (2.0 / (fi + fo)) ** 0.5
        if name.startswith("mp") and name.split(".")[-1] == last_mp:
            scale *= 0.1
        params[name + ".w"] = rng.standard_normal((fi, fo)) * scale
        params[name + ".b"] = np.zeros(fo)
    for name in _ln_stacks(hyper):  # LayerNorm: unit gain, zero shift (no RNG draws)
        params[name + ".ln.g"] = np.ones(FEATURE_WIDTH)
        params[name + ".ln.b"] = np.zeros(FEATURE_WIDTH)
    return GnnModel(hyper, params)


def _validate_params(model: GnnModel, width: int | None = None) -> None:
    expected = {}
    for name, fi, fo in _layer_specs(model.hyper, width):
        expected[name + ".w"] = (fi, fo)
        expected[name + ".b"] = (fo,)
    f = FEATURE_WIDTH if width is None else width
    for name in _ln_stacks(model.hyper):
        expected[name + ".ln.g"] = (f,)
        expected[name + ".ln.b"] = (f,)
    got = {k: np.shape(v) for k, v in model.params.items()}
    if got != expected:
        missing = sorted(set(expected) - set(got))
        extra = sorted(set(got) - set(expected))
        wrong = sorted(k for k in set(got) & set(expected) if got[k] != expected[k])
        raise DimensionMismatchError(
            f"parameter set does not match hyperparameters "
            f"(missing={missing}, unexpected={extra}, wrong shape={wrong})")
    for k, v in model.params.items():
        if not np.all(np.isfinite(v)):
            raise DataFormatError(f"non-finite weights in {k}")


# ---------------------------------------------------------------------------
# forward / factor (gnn.py:227-318), on the device
# ---------------------------------------------------------------------------


def _mesh_device(model: GnnModel, A: SparseMatrixCsr, mesh):
    """(positions, boundary) of A's rows as device fp64 arrays."""
    torch = _torch()
    if mesh is None:
        raise DimensionMismatchError("north_star mode needs mesh=(positions (n, dim), boundary (n,))")
    pos, bnd = mesh
    pos = to_device(np.ascontiguousarray(np.asarray(pos, dtype=np.float64)) if not is_device(pos) else pos)
    bnd = to_device(np.ascontiguousarray(np.asarray(bnd, dtype=np.float64)) if not is_device(bnd) else bnd,
                    dtype=torch.float64)
    if tuple(pos.shape) != (A.n, model.hyper.dim) or tuple(bnd.shape) != (A.n,):
        raise DimensionMismatchError(f"mesh must give ({A.n}, {model.hyper.dim}) positions and ({A.n},) flags")
    return pos.contiguous(), bnd.contiguous()


def _gnn_device(model: GnnModel, A: SparseMatrixCsr, rhs, values=None, want_edges=False, want_x0=False,
                mesh=None):
    """Runs npcg_gnn_build_factor. rhs (n, B) on device; values (nnz, B) or
    None (shared A). Returns (S, D, B, batched_vals, edge_out, x0_out)."""
    torch = _torch()
    handle = model.device()
    pat = A.device_pattern(factor=True)
    B = rhs.shape[1]
    if values is None:
        vals, vb = A.device_values(), 0
    else:
        vals, vb = to_device(values), 1
    m, n = A.nnz, A.n
    S = torch.empty((max(m, 1), B), dtype=torch.float64, device="cuda")
    D = torch.empty((max(n, 1), B), dtype=torch.float64, device="cuda")
    E = torch.empty((max(m, 1), B), dtype=torch.float64, device="cuda") if want_edges else None
    X0 = (torch.empty((max(n, 1), B), dtype=torch.float64, device="cuda")
          if want_x0 and model.hyper.with_x0_head else None)
    piv = ctypes.c_int64(-1)
    if model.hyper.north_star:
        pos, bnd = _mesh_device(model, A, mesh)
        rc = _native.lib().npcg_gnn_build_factor_mesh(handle.h, pat.handle, B, _native.ptr(vals), vb,
                                                      _native.ptr(rhs), _native.ptr(pos), _native.ptr(bnd),
                                                      _native.ptr(S), _native.ptr(D), _native.ptr(E),
                                                      ctypes.byref(piv), _native.stream_handle())
    else:
        rc = _native.lib().npcg_gnn_build_factor(handle.h, pat.handle, B, _native.ptr(vals), vb,
                                                 _native.ptr(rhs), _native.ptr(S), _native.ptr(D),
                                                 _native.ptr(E), _native.ptr(X0), ctypes.byref(piv),
                                                 _native.stream_handle())
    _native.check(rc, pivot=int(piv.value))
    return pat, S, D, E, X0


def run(model: GnnModel, graph: GraphData):
    """Inference (gnn.py:266-270): (edge scalars [m], node scalars [n] | None)."""
    A = graph.matrix
    if A is None:
        raise DimensionMismatchError("graph was not built by graph_from_system")
    rhs = to_device(graph.node_features[:, 0]).view(A.n, 1)
    _, _, _, E, X0 = _gnn_device(model, A, rhs, want_edges=True, want_x0=True)
    edges = E[: A.nnz, 0].cpu().numpy()
    x0 = X0[: A.n, 0].cpu().numpy() if X0 is not None else None
    return edges, x0


def lower_edge_indices(graph: GraphData) -> np.ndarray:
    return np.flatnonzero(graph.edge_src > graph.edge_dst)


def symmetrize_triangulate(edge_scalars, graph: GraphData):
    """0.5 (M[e] + M[pair(e)]) on strictly-lower edges (gnn.py:284-296)."""
    idx = lower_edge_indices(graph)
    rev = graph.edge_pair_index[idx]
    edge_scalars = np.asarray(edge_scalars, dtype=np.float64)
    return 0.5 * (edge_scalars[idx] + edge_scalars[rev])


def assemble_preconditioner(lower_values, A: SparseMatrixCsr) -> FactorPreconditioner:
    """P = (I + L') diag(A) (I + L')^T from strict-lower values in
    A.strict_lower() order (gnn.py:299-311); the factor is placed on A's
    pattern on the device."""
    d = A.diagonal()
    if np.any(d <= 0.0):
        bad = int(np.argmax(d <= 0.0))
        raise NotSpdError(f"nonpositive diagonal entry at row {bad}", pivot=bad)
    pattern = A.strict_lower()
    lower_values = np.asarray(lower_values, dtype=np.float64)
    if lower_values.shape != (pattern.nnz,):
        raise DimensionMismatchError(
            f"expected {pattern.nnz} lower-triangle values, got {lower_values.shape}")
    lf = LowerFactor(A.n, SparseMatrixCsr(A.n, pattern.row_ptr, pattern.col_idx, lower_values), d.copy())
    return FactorPreconditioner("learned", lf)


def build_learned(model: GnnModel, A: SparseMatrixCsr, b, mesh=None) -> FactorPreconditioner:
    """graph -> forward -> symmetrize -> assemble, end to end on the device
    (gnn.py:314-318). ``b`` may be numpy or a CUDA tensor. ``mesh`` =
    (positions (n, dim), boundary flags (n,)) of A's rows: required by the
    north_star mode (BASELINE.json's build(mesh, A, b, weights)), ignored by
    the reference network."""
    if tuple(b.shape) != (A.n,):
        raise DimensionMismatchError(f"b has shape {tuple(b.shape)}, expected ({A.n},)")
    return build_learned_batch(model, A, to_device(b).view(A.n, 1), mesh=mesh)


def build_learned_batch(model: GnnModel, A: SparseMatrixCsr, rhs, values=None, mesh=None) -> FactorPreconditioner:
    """B factors at once: rhs (n, B); ``values`` (nnz, B) for B distinct
    matrices on A's pattern (None: all share A); ``mesh`` shared by the
    batch (north_star mode). Returns one batched FactorPreconditioner
    (batch = B)."""
    rhs = to_device(rhs)
    if rhs.dim() != 2 or rhs.shape[0] != A.n:
        raise DimensionMismatchError("rhs must be (n, B)")
    B = rhs.shape[1]
    if B > _native.MAX_BATCH:
        raise DimensionMismatchError(f"batch must be <= {_native.MAX_BATCH}")
    if values is None:
        _check_values_symmetric(A, None)
    else:
        _check_values_symmetric(A, values)
    pat, S, D, _, _ = _gnn_device(model, A, rhs, values=values, mesh=mesh)
    lp = _lower_pattern(A)
    sb = B > 1
    Sv = S.view(-1) if sb else S[:, 0].contiguous()
    Dv = D.view(-1) if sb else D[:, 0].contiguous()
    return FactorPreconditioner("learned", None, device=(pat, Sv, sb, Dv, sb, B, A.n), lower_pattern=lp)


def _check_values_symmetric(A, values):
    pat = A.device_pattern(factor=True)  # DataFormatError: missing diagonal / asymmetric pattern
    if values is None:
        if not A.is_symmetric():
            raise DataFormatError("matrix values are not symmetric")
        return
    v = to_device(values)
    B = v.shape[1]
    ok = (ctypes.c_int32 * B)()
    _native.check(_native.lib().npcg_check_symmetric_values(pat.handle, B, _native.ptr(v), 1, ok,
                                                            _native.stream_handle()))
    if not all(ok):
        raise DataFormatError("matrix values are not symmetric")


_LOWER_PATTERNS = {}


def _lower_pattern(A: SparseMatrixCsr) -> SparseMatrixCsr:
    key = (id(A.row_ptr), id(A.col_idx))
    hit = _LOWER_PATTERNS.get(key)
    if hit is None or hit[0] is not A.row_ptr:
        rows = A.row_indices()
        keep = rows > A.col_idx
        sl = SparseMatrixCsr.from_coo(A.n, rows[keep], A.col_idx[keep], np.zeros(int(keep.sum())))
        hit = (A.row_ptr, A.col_idx, sl)
        _LOWER_PATTERNS[key] = hit
    return hit[2]


def predict_x0(model: GnnModel, graph: GraphData) -> np.ndarray:
    if not model.hyper.with_x0_head:
        raise PcgkitError("model has no x0 prediction head")
    _, x0 = run(model, graph)
    return x0


# ---------------------------------------------------------------------------
# checkpoints (gnn.py:335-374): byte-identical format
# ---------------------------------------------------------------------------


def save_model(path, model: GnnModel) -> None:
    """Reference checkpoints (format_version 1) are byte-identical to
    pcgkit's; north_star models write format_version 2 (their hyper-
    parameters add "mode" and "dim")."""
    _validate_params(model, model.width)
    hyper = {
        "l": model.hyper.l, "h": model.hyper.h, "n_mp": model.hyper.n_mp,
        "l_mp": model.hyper.l_mp, "h_mp": model.hyper.h_mp,
        "with_x0_head": model.hyper.with_x0_head, "normalize": model.hyper.normalize,
    }
    version = CHECKPOINT_VERSION
    if model.hyper.north_star:
        hyper.update(mode=model.hyper.mode, dim=model.hyper.dim)
        version = 2
    hyper = json.dumps(hyper, sort_keys=True)
    chunks = [f'{{"format_version": {version}, "hyper": {hyper}, "tensors": {{']
    for k, (name, arr) in enumerate(sorted(model.params.items())):
        data = ", ".join(format(x, ".17g") for x in np.asarray(arr).ravel())
        chunks.append(f'{", " if k else ""}{json.dumps(name)}: '
                      f'{{"data": [{data}], "shape": {json.dumps(list(np.shape(arr)))}}}')
    chunks.append("}}\n")
    with open(path, "w", encoding="ascii", newline="\n") as fh:
        fh.write("".join(chunks))


def load_model(path) -> GnnModel:
    try:
        with open(path, encoding="ascii") as fh:
            doc = json.load(fh)
    except (OSError, json.JSONDecodeError) as exc:
        raise DataFormatError(f"cannot read checkpoint {path}: {exc}") from exc
    version = doc.get("format_version")
    if version not in (CHECKPOINT_VERSION, 2):
        raise DataFormatError("unsupported checkpoint format version")
    if version == CHECKPOINT_VERSION and ("mode" in doc.get("hyper", {}) or "dim" in doc.get("hyper", {})):
        raise DataFormatError("format_version 1 checkpoints carry the reference network only")
    try:
        hyper = GnnHyperParams(**doc["hyper"])
        params = {name: np.array(rec["data"], dtype=np.float64).reshape(rec["shape"])
                  for name, rec in doc["tensors"].items()}
    except (KeyError, TypeError, ValueError) as exc:
        raise DataFormatError(f"malformed checkpoint: {exc}") from exc
    model = GnnModel(hyper, params)
    try:
        width = model.width
    except KeyError as exc:
        raise DimensionMismatchError(f"checkpoint lacks {exc}") from exc
    _validate_params(model, width)
    return model
