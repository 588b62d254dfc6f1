"""GPU parity of the elementary kernels against the oracle (bitwise where
the arithmetic contract promises it: per-row sums in the reference order,
unfused fp64, sparse.py:213-239)."""
import numpy as np
import pytest

from oracle import port
from paper_2305_16432_b200 import inputs, sparse

pytestmark = pytest.mark.gpu


def _ocsr(A):
    return port.Csr(A.n, A.row_ptr, A.col_idx, A.values)


def _heat(k=16, seed_cfg=1):
    return inputs.heat_2d(k=k, cfg=seed_cfg)


def test_spmv_bitwise(gpu):
    prob = _heat(24)
    A = prob.A
    x = np.random.default_rng(0).standard_normal(A.n)
    y = sparse.spmv(A, x)
    np.testing.assert_array_equal(y, port.spmv(_ocsr(A), x))


def test_spmv_batched_bitwise(gpu):
    import torch
    prob = _heat(20)
    A = prob.A
    rng = np.random.default_rng(1)
    for B in (1, 3, 8, 32, 64, 100, 128, 200, 256):  # 128+: four columns per lane
        X = rng.standard_normal((A.n, B))
        Y = sparse.spmv_device(A, torch.from_numpy(X).cuda(), B=B).cpu().numpy()
        for b in range(B):
            np.testing.assert_array_equal(Y[:, b], port.spmv(_ocsr(A), X[:, b]))


def test_apply_inverse_bitwise(gpu):
    prob = _heat(24)
    A = prob.A
    rng = np.random.default_rng(2)
    low = A.strict_lower()
    vals = rng.uniform(-0.3, 0.3, size=low.nnz)
    F = sparse.LowerFactor(A.n, sparse.SparseMatrixCsr(A.n, low.row_ptr, low.col_idx, vals), A.diagonal())
    r = rng.standard_normal(A.n)
    z = sparse.ldlt_apply_inverse(F, r)
    oF = port.Factor(A.n, port.Csr(A.n, low.row_ptr, low.col_idx, vals), A.diagonal())
    np.testing.assert_array_equal(z, oF.apply_inverse(r))


@pytest.mark.parametrize("chunk_rows", [None, "7", "64", "100000"])
def test_apply_inverse_chunkings_bitwise(gpu, monkeypatch, chunk_rows):
    """Every chunking of the schedule (one chunk, many small chunks,
    smem ring or not) gives the reference's bits."""
    if chunk_rows:
        monkeypatch.setenv("NPCG_CHUNK_ROWS", chunk_rows)
    prob = _heat(30)
    A = prob.A
    rng = np.random.default_rng(3)
    low = A.strict_lower()
    vals = rng.uniform(-0.4, 0.4, size=low.nnz)
    F = sparse.LowerFactor(A.n, sparse.SparseMatrixCsr(A.n, low.row_ptr, low.col_idx, vals), A.diagonal())
    r = rng.standard_normal(A.n)
    oF = port.Factor(A.n, port.Csr(A.n, low.row_ptr, low.col_idx, vals), A.diagonal())
    np.testing.assert_array_equal(sparse.ldlt_apply_inverse(F, r), oF.apply_inverse(r))


@pytest.mark.parametrize("path,k", [("lines", 26), ("lines", 64), ("lines", 96), ("levels", 27)])
def test_apply_inverse_paths_bitwise(gpu, monkeypatch, path, k):
    """Both triangular-solve engines -- the line wavefront (line-order
    vectors) and the chunked level schedule -- give the reference's bits,
    for a batch of systems sharing one factor and for per-system factors."""
    import torch
    if path == "levels":
        monkeypatch.setenv("NPCG_NO_LINES", "1")
    prob = _heat(k)
    A = prob.A
    rng = np.random.default_rng(4)
    low = A.strict_lower()
    B = 5
    vals = rng.uniform(-0.4, 0.4, size=(low.nnz, B))
    R = rng.standard_normal((A.n, B))
    pat = A.device_pattern(factor=True)
    # S on A's pattern (both triangles), per system: S[p * B + b]
    import paper_2305_16432_b200._native as nat
    S = torch.zeros((A.nnz, B), dtype=torch.float64, device="cuda")
    low_d = torch.from_numpy(vals).cuda().contiguous()
    nat.check(nat.lib().npcg_factor_from_lower(pat.handle, B, nat.ptr(low_d), 1, nat.ptr(S), nat.stream_handle()))
    D = torch.from_numpy(A.diagonal()).cuda()
    Z = sparse.apply_inverse_device(pat, S, True, D, False, torch.from_numpy(R).cuda(), B).cpu().numpy()
    for b in range(B):
        oF = port.Factor(A.n, port.Csr(A.n, low.row_ptr, low.col_idx, vals[:, b]), A.diagonal())
        np.testing.assert_array_equal(Z[:, b], oF.apply_inverse(R[:, b]))


@pytest.mark.parametrize("kr,k,B", [(2, 64, 8), (4, 64, 8), (2, 96, 6), (4, 200, 4), (2, 256, 4)])
def test_apply_inverse_several_rhs_per_cluster_bitwise(gpu, monkeypatch, kr, k, B):
    """NPCG_LINE_KR right-hand sides per cluster (shared factor: one staged
    factor, interleaved dependency chains in the line warp) give the
    reference's bits for every column."""
    import torch
    monkeypatch.setenv("NPCG_LINE_KR", str(kr))
    prob = _heat(k)
    A = prob.A
    rng = np.random.default_rng(40 + kr)
    low = A.strict_lower()
    vals = rng.uniform(-0.4, 0.4, size=low.nnz)
    R = rng.standard_normal((A.n, B))
    pat = A.device_pattern(factor=True)
    import paper_2305_16432_b200._native as nat
    S = torch.zeros((A.nnz,), dtype=torch.float64, device="cuda")
    low_d = torch.from_numpy(vals).cuda().contiguous()
    nat.check(nat.lib().npcg_factor_from_lower(pat.handle, 1, nat.ptr(low_d), 0, nat.ptr(S), nat.stream_handle()))
    D = torch.from_numpy(A.diagonal()).cuda()
    Z = sparse.apply_inverse_device(pat, S, False, D, False, torch.from_numpy(R).cuda(), B).cpu().numpy()
    oF = port.Factor(A.n, port.Csr(A.n, low.row_ptr, low.col_idx, vals), A.diagonal())
    for b in range(B):
        np.testing.assert_array_equal(Z[:, b], oF.apply_inverse(R[:, b]))


def test_pcg_several_rhs_per_cluster_same_iterates(gpu, monkeypatch):
    """A shared-factor batch solved with 1, 2 and 4 right-hand sides per
    cluster: same iteration counts and bitwise equal solutions (same launch
    shape otherwise), including columns that converge at different passes."""
    import torch
    from paper_2305_16432_b200 import gnn, pcg
    outs = []
    for kr in ("1", "2", "4"):
        monkeypatch.setenv("NPCG_LINE_KR", kr)
        # the same stage length for every kr (the shared-memory budget would pick longer
        # stages for kr = 1): dot products then accumulate in the same order
        monkeypatch.setenv("NPCG_LINE_CFG", str(1 * 16 + 4))
        prob = inputs.poisson_2d(k=96, batch=8)  # 95 lines: one CTA per cluster for every kr
        A = prob.A
        rng = np.random.default_rng(7)
        P = gnn.assemble_preconditioner(rng.uniform(-0.2, 0.2, A.strict_lower().nnz), A)
        rhs = prob.rhs.copy()
        rhs[:, 3] = 0.0  # a zero right-hand side inside the batch
        rhs[:, 5] *= 1e-3
        X, reps = pcg.pcg_solve_batch(A, torch.from_numpy(rhs).cuda(), P,
                                      pcg.SolveOptions(thresholds=(1e-4, 1e-10), max_iter=2000))
        outs.append((X.cpu().numpy(), [r.iterations for r in reps], [r.converged for r in reps]))
    assert all(outs[0][2])
    assert len(set(outs[0][1])) > 1  # columns finish at different passes
    for X, its, conv in outs[1:]:
        assert its == outs[0][1] and conv == outs[0][2]
        np.testing.assert_array_equal(X, outs[0][0])


def test_apply_inverse_wide_grid_bitwise(gpu):
    """A 513 x 513 grid (511 lines: 16 warps, a 2-CTA cluster per system,
    one-tile stages): bitwise equal to the reference's solve."""
    prob = inputs.poisson_2d(k=512, batch=1)
    A = prob.A
    rng = np.random.default_rng(5)
    low = A.strict_lower()
    vals = rng.uniform(-0.3, 0.3, size=low.nnz)
    F = sparse.LowerFactor(A.n, sparse.SparseMatrixCsr(A.n, low.row_ptr, low.col_idx, vals), A.diagonal())
    R = rng.standard_normal((A.n, 2))
    oF = port.Factor(A.n, port.Csr(A.n, low.row_ptr, low.col_idx, vals), A.diagonal())
    for b in range(2):
        np.testing.assert_array_equal(sparse.ldlt_apply_inverse(F, R[:, b]), oF.apply_inverse(R[:, b]))


_LINES_VS_LEVELS = r"""
import os, sys, numpy as np, torch
sys.path.insert(0, os.environ["REPO"])
from paper_2305_16432_b200 import gnn, inputs, pcg
gnn.FEATURE_WIDTH = 64
prob = inputs.poisson_2d(k=256, batch=64)
model = gnn.create_model(gnn.GnnHyperParams(l=1, h=64, n_mp=2, l_mp=1, h_mp=64), seed=3)
for r in range(2):
    for s in ("node", "edge"):
        model.params[f"mp{r}.{s}.1.w"] *= 10.0
rhs = torch.from_numpy(prob.rhs).cuda()
P = gnn.build_learned(model, prob.A, rhs[:, 0])
X, reps = pcg.pcg_solve_batch(prob.A, rhs, P, pcg.SolveOptions(thresholds=(1e-8,), max_iter=3000))
np.save(os.environ["OUT"], np.concatenate([np.array([[r.iterations for r in reps]], float), X.cpu().numpy()]))
"""


def test_pcg_line_path_matches_level_path(gpu, tmp_path):
    """Config-1-sized PCG with a GNN factor (B = 64, shared L'): the
    line-order path converges like the level path -- iterations within
    +-3, solutions within 1e-8 -- after GNN kernels have left arbitrary
    bits in shared memory (staged padding slots must not reach the dot
    products)."""
    import os
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "run.py"
    script.write_text(_LINES_VS_LEVELS)
    out = {}
    for path in ("lines", "levels"):
        env = dict(os.environ, REPO=repo, OUT=str(tmp_path / f"{path}.npy"))
        if path == "levels":
            env["NPCG_NO_LINES"] = "1"
        subprocess.run([sys.executable, str(script)], env=env, check=True, timeout=600)
        out[path] = np.load(tmp_path / f"{path}.npy")
    it_l, it_v = out["lines"][0], out["levels"][0]
    assert it_l.max() < 3000 and it_v.max() < 3000
    assert np.abs(it_l - it_v).max() <= 3
    xl, xv = out["lines"][1:], out["levels"][1:]
    rel = np.abs(xl - xv).max(axis=0) / np.abs(xv).max(axis=0)
    assert rel.max() < 1e-8


def test_pcg_line_path_reproducible(gpu):
    """A few PCG iterations through the line-order path are bitwise
    reproducible, also right after GNN kernels have left arbitrary bits in
    shared memory (padding slots of the staged vectors must never carry
    stale data into the dot products)."""
    import torch
    from paper_2305_16432_b200 import gnn, pcg
    old_width = gnn.FEATURE_WIDTH
    try:
        gnn.FEATURE_WIDTH = 64
        prob = inputs.poisson_2d(k=256, batch=64)
        A = prob.A
        model = gnn.create_model(gnn.GnnHyperParams(l=1, h=64, n_mp=2, l_mp=1, h_mp=64), seed=3)
        rhs = torch.from_numpy(prob.rhs).cuda()
        outs = []
        for _ in range(3):
            P = gnn.build_learned(model, A, rhs[:, 0])
            X, _ = pcg.pcg_solve_batch(A, rhs, P, pcg.SolveOptions(thresholds=(1e-14,), max_iter=4))
            outs.append(X.cpu().numpy().view(np.int64).copy())
    finally:
        gnn.FEATURE_WIDTH = old_width
    for o in outs[1:]:
        np.testing.assert_array_equal(o, outs[0])
