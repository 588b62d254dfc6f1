"""Seeded synthetic inputs for the BASELINE.json configs (input generation,
not the solve path).

The reference ships P1 FEM assembly (pkg/src/pcgkit/fem.py:42-215) as a
per-element Python loop over unjittered grids (mesh.py:149-178). The
configs need jittered grids, per-element coefficients and random-field
right-hand sides, so this module generates them, vectorised in numpy.
The arithmetic per element and the scatter order follow fem.py:42-69 and
fem.py:116-134 exactly (COO in element order, lexsort + reduceat), so the
assembled matrices are bitwise symmetric -- graph_from_system requires it
(gnn.py:79-82) -- and, on the same vertices, bitwise equal to the
reference's own assembly (pinned in tests/test_inputs.py against goldens
produced by pcgkit.fem).

Seeds: np.random.SeedSequence(1000 * cfg + 17).spawn(B), one stream per
system / right-hand side; draws in the order jitter, coefficients, RHS.
Random fields use random Fourier features (squared-exponential
covariance): f(x) = sqrt(2/R) sum_r cos(w_r . x + phi_r), w ~ N(0, l^-2 I).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .sparse import SparseMatrixCsr

MASS_TEMPLATE = np.array([[2.0, 1.0, 1.0], [1.0, 2.0, 1.0], [1.0, 1.0, 2.0]]) / 12.0
GRF_FEATURES = 64


@dataclass
class Mesh2D:
    vertices: np.ndarray   # (nv, 2)
    triangles: np.ndarray  # (nt, 3) counter-clockwise
    boundary: np.ndarray   # (nv,) bool


def unit_square(k: int, jitter: float = 0.0, rng: np.random.Generator | None = None) -> Mesh2D:
    """(k+1)^2 vertices, cells split along the (1,1) diagonal, vertex and
    triangle order of mesh.generate_unit_square (mesh.py:149-178); interior
    vertices moved by U[-jitter, jitter] * h per coordinate."""
    axis = np.arange(k + 1) / k
    xs, ys = np.meshgrid(axis, axis, indexing="xy")
    v = np.column_stack([xs.ravel(), ys.ravel()])
    boundary = ((xs == 0.0) | (xs == 1.0) | (ys == 0.0) | (ys == 1.0)).ravel()
    if jitter > 0.0:
        inner = np.flatnonzero(~boundary)
        v[inner] += rng.uniform(-1.0, 1.0, size=(len(inner), 2)) * (jitter / k)
    ix, iy = np.meshgrid(np.arange(k), np.arange(k), indexing="xy")
    a = (iy * (k + 1) + ix).ravel()
    b, c, d = a + 1, a + k + 2, a + k + 1
    tris = np.empty((2 * k * k, 3), dtype=np.int64)
    tris[0::2] = np.column_stack([a, b, c])
    tris[1::2] = np.column_stack([a, c, d])
    return Mesh2D(v, tris, boundary)


def element_blocks(mesh: Mesh2D):
    """Per-element 3x3 stiffness and mass blocks, (nt, 3, 3) each, with the
    operation order of fem.element_stiffness / element_mass."""
    p = mesh.vertices[mesh.triangles]
    twice = (p[:, 1, 0] - p[:, 0, 0]) * (p[:, 2, 1] - p[:, 0, 1]) - \
        (p[:, 1, 1] - p[:, 0, 1]) * (p[:, 2, 0] - p[:, 0, 0])
    if np.any(twice <= 0.0):
        raise ValueError("degenerate or clockwise triangle (reduce the jitter)")
    bs = np.stack([p[:, 1, 1] - p[:, 2, 1], p[:, 2, 1] - p[:, 0, 1], p[:, 0, 1] - p[:, 1, 1]], axis=1)
    cs = np.stack([p[:, 2, 0] - p[:, 1, 0], p[:, 0, 0] - p[:, 2, 0], p[:, 1, 0] - p[:, 0, 0]], axis=1)
    K = (bs[:, :, None] * bs[:, None, :] + cs[:, :, None] * cs[:, None, :]) / (2.0 * np.abs(twice))[:, None, None]
    M = (np.abs(twice) / 2.0)[:, None, None] * MASS_TEMPLATE[None]
    return K, M


class Assembler:
    """Scatter of per-element blocks into the fixed CSR pattern, in element
    order (fem.py:116-134); the sort is computed once per mesh."""

    def __init__(self, n_vertices: int, triangles: np.ndarray):
        npe = triangles.shape[1]  # 3 (triangles) or 4 (tetrahedra)
        rows = np.repeat(triangles, npe, axis=1).ravel()
        cols = np.tile(triangles, (1, npe)).ravel()
        order = np.lexsort((cols, rows))
        r, c = rows[order], cols[order]
        head = np.ones(len(r), dtype=bool)
        head[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
        self.order = order
        self.starts = np.flatnonzero(head)
        self.n = n_vertices
        self.row_ptr = np.zeros(n_vertices + 1, dtype=np.int64)
        np.cumsum(np.bincount(r[self.starts], minlength=n_vertices), out=self.row_ptr[1:])
        self.col_idx = np.ascontiguousarray(c[self.starts])

    def values(self, blocks: np.ndarray) -> np.ndarray:
        return np.add.reduceat(blocks.reshape(-1)[self.order], self.starts)

    def matrix(self, values) -> SparseMatrixCsr:
        return SparseMatrixCsr(self.n, self.row_ptr, self.col_idx, values)


class Restriction:
    """Symmetric restriction to free vertices (SparseMatrixCsr.submatrix,
    sparse.py:155-163), precomputed once per (pattern, free set)."""

    def __init__(self, A: SparseMatrixCsr, free: np.ndarray):
        remap = -np.ones(A.n, dtype=np.int64)
        remap[free] = np.arange(len(free), dtype=np.int64)
        rows = remap[A.row_indices()]
        cols = remap[A.col_idx]
        self.sel = np.flatnonzero((rows >= 0) & (cols >= 0))
        # rows stay sorted by (row, col) after restriction: no duplicates possible
        rr, cc = rows[self.sel], cols[self.sel]
        self.free = free
        self.n = len(free)
        self.row_ptr = np.zeros(self.n + 1, dtype=np.int64)
        np.cumsum(np.bincount(rr, minlength=self.n), out=self.row_ptr[1:])
        self.col_idx = np.ascontiguousarray(cc)

    def matrix(self, values_full) -> SparseMatrixCsr:
        return SparseMatrixCsr(self.n, self.row_ptr, self.col_idx, np.ascontiguousarray(values_full[self.sel]))


def grf_2d(points: np.ndarray, rng: np.random.Generator, length: float, n_features: int = GRF_FEATURES):
    """Squared-exponential Gaussian random field sampled at points (RFF)."""
    w = rng.standard_normal((n_features, points.shape[1])) / length
    phi = rng.uniform(0.0, 2.0 * np.pi, size=n_features)
    # phases in float32: the field is a random input, not a checked quantity
    ph = (points @ w.T + phi).astype(np.float32)
    return np.sqrt(2.0 / n_features) * np.cos(ph).sum(axis=1, dtype=np.float64)


def gaussian_bumps(points: np.ndarray, rng: np.random.Generator, count=8, width=(0.05, 0.2)):
    centers = rng.uniform(0.0, 1.0, size=(count, 2))
    widths = rng.uniform(width[0], width[1], size=count)
    amps = rng.standard_normal(count)
    d2 = ((points[:, None, :] - centers[None, :, :]) ** 2).sum(axis=2)
    return (amps[None, :] * np.exp(-d2 / (2.0 * widths[None, :] ** 2))).sum(axis=1)


def streams(cfg: int, count: int):
    return [np.random.default_rng(s) for s in np.random.SeedSequence(1000 * cfg + 17).spawn(count)]


# ---------------------------------------------------------------------------
# configs (BASELINE.json "configs")
# ---------------------------------------------------------------------------


@dataclass
class Problem:
    name: str
    A: SparseMatrixCsr         # shared pattern (values of system 0)
    rhs: np.ndarray            # (n, B)
    values: np.ndarray | None  # (nnz, B) for distinct systems, else None
    rtol: float
    max_iter: int | None
    meta: dict
    # north_star GNN inputs for the rows of A: positions (n, dim) and the
    # boundary flag (domain boundary, or next to an eliminated Dirichlet node)
    geometry: tuple | None = None
    # what DeviceAssembler needs to form `values` on the device instead of uploading them:
    # {"elements", "vertices", "coef" (n_elements, B), "mode", "scale"} (distinct-system configs)
    assembly: dict | None = None


def _free_geometry(mesh, full_pattern: SparseMatrixCsr, free: np.ndarray):
    """Positions of the free rows and their flag: adjacent to a Dirichlet
    (eliminated) node through the assembled pattern."""
    rows = full_pattern.row_indices()
    touch = np.zeros(full_pattern.n, dtype=bool)
    np.logical_or.at(touch, rows, mesh.boundary[full_pattern.col_idx])
    return np.ascontiguousarray(mesh.vertices[free]), touch[free]


def heat_2d(k=32, jitter=0.2, dt=1e-2, alpha=1.0, cfg=1, batch=1) -> Problem:
    """Config 1: heat step A = M + dt*alpha*K on a jittered k x k square, no
    Dirichlet rows (n = (k+1)^2); b = M u0, u0 = 8 Gaussian bumps."""
    rngs = streams(cfg, batch)
    vals, rhs = [], []
    A0 = None
    for rng in rngs:
        mesh = unit_square(k, jitter, rng)
        K, M = element_blocks(mesh)
        asm = Assembler(len(mesh.vertices), mesh.triangles)
        Kv, Mv = asm.values(K), asm.values(M)
        A = asm.matrix(Mv + (dt * alpha) * Kv)
        Mm = asm.matrix(Mv)
        u0 = gaussian_bumps(mesh.vertices, rng)
        b = _host_spmv(Mm, u0)
        A0 = A0 or A
        vals.append(A.values)
        rhs.append(b)
    values = None if batch == 1 else np.stack(vals, axis=1)
    if values is not None:
        A0 = A0.with_values(values[:, 0].copy())
    return Problem("heat2d", A0, np.stack(rhs, axis=1), values, 1e-8, 2000,
                   {"k": k, "jitter": jitter, "dt": dt, "cfg": cfg},
                   (np.ascontiguousarray(mesh.vertices), mesh.boundary.copy()))


def poisson_2d(k=256, jitter=0.2, batch=64, cfg=2, first=0) -> Problem:
    """Config 2: Poisson stiffness on a jittered k x k square, full-boundary
    Dirichlet eliminated (n = (k-1)^2); B right-hand sides (M f)[free], f a
    squared-exponential GRF with length scale U[0.05, 0.3]. ``first`` skips
    that many RHS streams (one batch per rank); the mesh is always the one
    drawn from stream 0."""
    rngs = streams(cfg, first + batch)[first:]
    mesh_rng = rngs[0] if first == 0 else streams(cfg, 1)[0]
    mesh = unit_square(k, jitter, mesh_rng)  # one shared mesh (one L' for all RHS)
    K, M = element_blocks(mesh)
    asm = Assembler(len(mesh.vertices), mesh.triangles)
    Kv, Mv = asm.values(K), asm.values(M)
    free = np.flatnonzero(~mesh.boundary)
    red = Restriction(asm.matrix(Kv), free)
    A = red.matrix(Kv)
    Mm = asm.matrix(Mv)
    rhs = np.empty((len(free), batch))
    for j, rng in enumerate(rngs):
        f = grf_2d(mesh.vertices, rng, rng.uniform(0.05, 0.3))
        rhs[:, j] = _host_spmv(Mm, f)[free]
    return Problem("poisson2d", A, rhs, None, 1e-8, None, {"k": k, "jitter": jitter, "cfg": cfg},
                   _free_geometry(mesh, asm.matrix(Kv), free))


def wave_2d(k=512, jitter=0.2, dt=1e-3, sigma=0.5, batch=32, cfg=3, first=0) -> Problem:
    """Config 3: implicit wave step A = M + dt^2 K_c, c = exp(sigma * GRF) per
    element; b = M g with g a GRF; distinct A per system, one shared mesh
    topology (jitter drawn from the config stream, shared)."""
    rngs = streams(cfg, first + batch)[first:]
    mesh = unit_square(k, jitter, np.random.default_rng(np.random.SeedSequence(1000 * cfg + 17).entropy))
    K, M = element_blocks(mesh)
    asm = Assembler(len(mesh.vertices), mesh.triangles)
    Mv = asm.values(M)
    Mm = asm.matrix(Mv)
    cent = mesh.vertices[mesh.triangles].mean(axis=1)
    vals = np.empty((len(asm.col_idx), batch))
    rhs = np.empty((len(mesh.vertices), batch))
    coef = np.empty((len(mesh.triangles), batch))
    for j, rng in enumerate(rngs):
        c = np.exp(sigma * grf_2d(cent, rng, rng.uniform(0.05, 0.3)))
        Kc = asm.values(K * c[:, None, None])
        vals[:, j] = Mv + (dt * dt) * Kc
        coef[:, j] = c
        rhs[:, j] = _host_spmv(Mm, grf_2d(mesh.vertices, rng, rng.uniform(0.05, 0.3)))
    A = asm.matrix(np.ascontiguousarray(vals[:, 0]))
    return Problem("wave2d", A, rhs, vals, 1e-8, None, {"k": k, "jitter": jitter, "dt": dt, "cfg": cfg},
                   (np.ascontiguousarray(mesh.vertices), mesh.boundary.copy()),
                   {"elements": mesh.triangles, "vertices": mesh.vertices, "coef": coef, "mode": "M+sK",
                    "scale": dt * dt})


# ---------------------------------------------------------------------------
# 3-D inputs (configs 4 and 5): Kuhn-split unit cube, P1 tetrahedra. The
# reference has no 3-D FEM; this restates P1 on tetrahedra in the 2-D code's
# style (element blocks in a fixed elementwise operation order, the same
# COO lexsort / reduceat scatter), so assembled matrices are bitwise
# symmetric as graph_from_system requires (gnn.py:79-82).
# ---------------------------------------------------------------------------


@dataclass
class Mesh3D:
    vertices: np.ndarray   # (nv, 3)
    tets: np.ndarray       # (nt, 4), positive orientation
    boundary: np.ndarray   # (nv,) bool


def unit_cube(k: int, jitter: float = 0.0, rng: np.random.Generator | None = None) -> Mesh3D:
    """(k+1)^3 vertices (x fastest), every cell split into the 6 Kuhn
    tetrahedra around its (0,0,0)-(1,1,1) diagonal; interior vertices moved by
    U[-jitter, jitter] * h per coordinate."""
    axis = np.arange(k + 1) / k
    zs, ys, xs = np.meshgrid(axis, axis, axis, indexing="ij")
    v = np.column_stack([xs.ravel(), ys.ravel(), zs.ravel()])
    boundary = ((v == 0.0) | (v == 1.0)).any(axis=1)
    if jitter > 0.0:
        inner = np.flatnonzero(~boundary)
        v[inner] += rng.uniform(-1.0, 1.0, size=(len(inner), 3)) * (jitter / k)
    n1 = k + 1
    step = np.array([1, n1, n1 * n1])
    iz, iy, ix = np.meshgrid(np.arange(k), np.arange(k), np.arange(k), indexing="ij")
    o = (iz * n1 * n1 + iy * n1 + ix).ravel()
    tets = []
    for perm, sign in (((0, 1, 2), 1), ((0, 2, 1), -1), ((1, 0, 2), -1), ((1, 2, 0), 1), ((2, 0, 1), 1),
                       ((2, 1, 0), -1)):
        a = o
        b = a + step[perm[0]]
        c = b + step[perm[1]]
        d = c + step[perm[2]]
        tets.append(np.column_stack([a, b, c, d] if sign > 0 else [a, c, b, d]))
    tets = np.stack(tets, axis=1).reshape(-1, 4).astype(np.int64)  # cell-major, 6 per cell
    return Mesh3D(v, tets, boundary)


def tet_blocks(mesh: Mesh3D):
    """Per-tetrahedron 4x4 P1 stiffness and mass blocks, (nt, 4, 4) each:
    K_ij = |T| grad l_i . grad l_j, M_ij = |T| (1 + d_ij) / 20."""
    p = mesh.vertices[mesh.tets]
    e1, e2, e3 = p[:, 1] - p[:, 0], p[:, 2] - p[:, 0], p[:, 3] - p[:, 0]
    c23, c31, c12 = np.cross(e2, e3), np.cross(e3, e1), np.cross(e1, e2)
    det = (e1[:, 0] * c23[:, 0] + e1[:, 1] * c23[:, 1]) + e1[:, 2] * c23[:, 2]
    if np.any(det <= 0.0):
        raise ValueError("degenerate or inverted tetrahedron (reduce the jitter)")
    g = np.empty((len(det), 4, 3))
    g[:, 1], g[:, 2], g[:, 3] = c23 / det[:, None], c31 / det[:, None], c12 / det[:, None]
    g[:, 0] = -((g[:, 1] + g[:, 2]) + g[:, 3])
    vol = det / 6.0
    dots = (g[:, :, None, 0] * g[:, None, :, 0] + g[:, :, None, 1] * g[:, None, :, 1]) + \
        g[:, :, None, 2] * g[:, None, :, 2]
    K = vol[:, None, None] * dots
    M = (vol / 20.0)[:, None, None] * (np.ones((4, 4)) + np.eye(4))[None]
    return K, M


def poisson_3d(k=64, jitter=0.15, batch=128, cfg=4, first=0) -> Problem:
    """Config 4: Poisson stiffness on a jittered Kuhn cube, full-boundary
    Dirichlet eliminated (n = (k-1)^3); B right-hand sides (M f)[free], f a
    3-D squared-exponential GRF with length scale U[0.05, 0.3]; one mesh."""
    rngs = streams(cfg, first + batch)[first:]
    mesh_rng = rngs[0] if first == 0 else streams(cfg, 1)[0]
    mesh = unit_cube(k, jitter, mesh_rng)
    K, M = tet_blocks(mesh)
    asm = Assembler(len(mesh.vertices), mesh.tets)
    Kv, Mv = asm.values(K), asm.values(M)
    free = np.flatnonzero(~mesh.boundary)
    red = Restriction(asm.matrix(Kv), free)
    A = red.matrix(Kv)
    Mm = asm.matrix(Mv)
    rhs = np.empty((len(free), batch))
    for j, rng in enumerate(rngs):
        f = grf_2d(mesh.vertices, rng, rng.uniform(0.05, 0.3))
        rhs[:, j] = _host_spmv(Mm, f)[free]
    return Problem("poisson3d", A, rhs, None, 1e-8, None, {"k": k, "jitter": jitter, "cfg": cfg},
                   _free_geometry(mesh, asm.matrix(Kv), free))


def heat_3d(k=128, jitter=0.15, dt=1e-3, sigma=1.0, batch=8, cfg=5, first=0) -> Problem:
    """Config 5: A = M + dt K_kappa on a jittered Kuhn cube (no Dirichlet rows,
    n = (k+1)^3), kappa = exp(sigma GRF) per element and system; b = M g with g
    a GRF; distinct A per system, one mesh (rtol 1e-10)."""
    rngs = streams(cfg, first + batch)[first:]
    mesh = unit_cube(k, jitter, np.random.default_rng(np.random.SeedSequence(1000 * cfg + 17).entropy))
    K, M = tet_blocks(mesh)
    asm = Assembler(len(mesh.vertices), mesh.tets)
    Mv = asm.values(M)
    Mm = asm.matrix(Mv)
    cent = mesh.vertices[mesh.tets].mean(axis=1)
    vals = np.empty((len(asm.col_idx), batch))
    rhs = np.empty((len(mesh.vertices), batch))
    for j, rng in enumerate(rngs):
        kap = np.exp(sigma * grf_2d(cent, rng, rng.uniform(0.05, 0.3)))
        vals[:, j] = Mv + dt * asm.values(K * kap[:, None, None])
        rhs[:, j] = _host_spmv(Mm, grf_2d(mesh.vertices, rng, rng.uniform(0.05, 0.3)))
    A = asm.matrix(np.ascontiguousarray(vals[:, 0]))
    return Problem("heat3d", A, rhs, vals, 1e-10, None, {"k": k, "jitter": jitter, "dt": dt, "cfg": cfg},
                   (np.ascontiguousarray(mesh.vertices), mesh.boundary.copy()))


def _host_spmv(A: SparseMatrixCsr, x):
    """Input-generation helper (not the solve path): y = A x in numpy, each
    row summed sequentially in stored order like sparse.py:213-219, so
    loads such as b = M u0 match the reference's assembly bitwise."""
    deg = np.diff(A.row_ptr)
    y = np.zeros(A.n)
    for k in range(int(deg.max()) if A.n else 0):
        rows = np.flatnonzero(deg > k)
        p = A.row_ptr[rows] + k
        y[rows] += A.values[p] * x[A.col_idx[p]]
    return y


class DeviceAssembler:
    """P1 assembly on the device (libnpcg ``npcg_fem_assemble``, csrc/fem.cu):
    the same element topology as :class:`Assembler` -- triangles (nt, 3) with
    2-D vertices or tetrahedra (nt, 4) with 3-D vertices -- any number of
    vertex sets / per-element coefficients per call, values bit-identical to
    ``Assembler.values(element_blocks(...))`` (fem.py:42-69, 116-134) and to
    ``Assembler.values(tet_blocks(...))``.

    ``values(vertices, coef=None, mode="K" | "M" | "M+sK", scale=1.0)``:
    vertices (nv, dim) or (nv, dim, B); coef None, (nt,) or (nt, B); returns a
    device float64 tensor (nnz,) or (nnz, B). Raises ValueError on a
    degenerate / negatively oriented element like element_blocks / tet_blocks."""

    MODES = {"K": 0, "M": 1, "M+sK": 2}

    def __init__(self, n_vertices: int, elements: np.ndarray):
        import ctypes

        from . import _native
        self._lib = _native.lib()
        tri = np.ascontiguousarray(elements, dtype=np.int64)
        if tri.ndim != 2 or tri.shape[1] not in (3, 4):
            raise ValueError("elements must be (nt, 3) triangles or (nt, 4) tetrahedra")
        self.dim = tri.shape[1] - 1
        h = ctypes.c_void_p()
        _native.check(self._lib.npcg_fem_plan_create_p1(int(n_vertices), len(tri), tri.shape[1], tri.ctypes.data,
                                                        ctypes.byref(h)))
        self._h = h
        nnz = ctypes.c_int64()
        _native.check(self._lib.npcg_fem_plan_pattern(h, ctypes.byref(nnz), None, None))
        self.n, self.nnz, self.n_triangles = int(n_vertices), int(nnz.value), len(tri)
        self.row_ptr = np.zeros(self.n + 1, dtype=np.int64)
        self.col_idx = np.zeros(self.nnz, dtype=np.int64)
        _native.check(self._lib.npcg_fem_plan_pattern(h, ctypes.byref(nnz), self.row_ptr.ctypes.data,
                                                      self.col_idx.ctypes.data))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.npcg_fem_plan_destroy(h)
            self._h = None

    def values(self, vertices, coef=None, mode: str = "K", scale: float = 1.0, check: bool = True):
        import torch

        from . import _native
        if mode not in self.MODES:
            raise ValueError(f"mode must be one of {sorted(self.MODES)}")
        V = torch.as_tensor(vertices, dtype=torch.float64, device="cuda").contiguous()
        if V.dim() not in (2, 3) or V.shape[0] != self.n or V.shape[1] != self.dim:
            raise ValueError(f"vertices must be (n_vertices, {self.dim}) or (n_vertices, {self.dim}, B)")
        B = V.shape[2] if V.dim() == 3 else 1
        C = None
        if coef is not None:
            C = torch.as_tensor(coef, dtype=torch.float64, device="cuda").contiguous()
            if C.shape[0] != self.n_triangles or C.dim() not in (1, 2):
                raise ValueError("coef must be (n_triangles,) or (n_triangles, B)")
            if C.dim() == 2:
                if B == 1:
                    B = C.shape[1]
                elif C.shape[1] != B:
                    raise ValueError("coef and vertices disagree on the batch")
        batched = V.dim() == 3 or (C is not None and C.dim() == 2)
        out = torch.empty((self.nnz, B) if batched else (self.nnz,), dtype=torch.float64, device="cuda")
        bad = torch.zeros(1, dtype=torch.int32, device="cuda")
        _native.check(self._lib.npcg_fem_assemble(
            self._h, B, _native.ptr(V), int(V.dim() == 3), _native.ptr(C), int(C is not None and C.dim() == 2),
            self.MODES[mode], float(scale), _native.ptr(out), _native.ptr(bad), _native.stream_handle()))
        if check and int(bad.item()):
            raise ValueError("degenerate or inverted element (reduce the jitter)")
        return out


class DeviceRestriction(Restriction):
    """:class:`Restriction` whose value gather runs on the device
    (``npcg_gather_values``): the Dirichlet elimination of fem.py:209-215
    applied to device-assembled values without a host round trip.
    ``values(full)`` takes a device tensor (nnz_full,) or (nnz_full, B)."""

    def values(self, values_full):
        import torch

        from . import _native
        if not hasattr(self, "_sel_dev"):
            self._sel_dev = torch.from_numpy(self.sel.astype(np.int32)).cuda()
        src = values_full.contiguous()
        batched = src.dim() == 2
        B = src.shape[1] if batched else 1
        out = torch.empty((len(self.sel), B) if batched else (len(self.sel),), dtype=torch.float64, device=src.device)
        _native.check(_native.lib().npcg_gather_values(len(self.sel), B, int(batched), _native.ptr(self._sel_dev),
                                                       _native.ptr(src), _native.ptr(out), _native.stream_handle()))
        return out
