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
    for B in (1, 3, 8, 32, 64, 100):
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
