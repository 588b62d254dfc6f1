"""Matrix Market exchange (paper_2305_16432_b200.mmio) against the
reference's own writer output (tests/golden/mmio_*.mtx, minted by
tests/golden/make_mmio_golden.py with pcgkit.mmio): byte-identical text,
bit-exact parsing, and the error cases of pkg/tests/test_mmio.py. CPU only."""
import os

import numpy as np
import pytest

from paper_2305_16432_b200 import inputs, mmio
from paper_2305_16432_b200.errors import DataFormatError
from paper_2305_16432_b200.sparse import SparseMatrixCsr

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def read(name):
    with open(os.path.join(GOLD, name)) as fh:
        return fh.read()


def same_matrix(a, b):
    assert a.n == b.n
    np.testing.assert_array_equal(a.row_ptr, b.row_ptr)
    np.testing.assert_array_equal(a.col_idx, b.col_idx)
    np.testing.assert_array_equal(a.values.view(np.int64), b.values.view(np.int64))


def test_writer_matches_reference_bytes():
    A = inputs.heat_2d(k=4).A
    assert mmio.matrix_to_text(A, symmetric=True) == read("mmio_heat4_symmetric.mtx")
    assert mmio.matrix_to_text(A, symmetric=False) == read("mmio_heat4_general.mtx")
    p = inputs.heat_2d(k=4)
    v = np.concatenate([p.rhs[:, 0], [1.0 / 3.0, -2.5e-308, 0.0, -0.0, 1e300]])
    assert mmio.vector_to_text(v) == read("mmio_heat4_rhs.mtx")


def test_reader_on_reference_files_is_exact():
    A = inputs.heat_2d(k=4).A
    same_matrix(mmio.matrix_from_text(read("mmio_heat4_symmetric.mtx")), A)
    same_matrix(mmio.matrix_from_text(read("mmio_heat4_general.mtx")), A)
    v = mmio.vector_from_text(read("mmio_heat4_rhs.mtx"))
    assert v.shape == (30,) and np.signbit(v[-2]) and v[-1] == 1e300


def test_symmetric_header_and_lower_triangle():
    text = mmio.matrix_to_text(SparseMatrixCsr.from_dense([[2.0, 1.0], [1.0, 3.0]]))
    lines = text.splitlines()
    assert lines[0] == "%%MatrixMarket matrix coordinate real symmetric"
    assert lines[1] == "2 2 3"


def test_general_keeps_asymmetry_and_symmetric_rejects_it():
    a = SparseMatrixCsr.from_dense([[1.0, 5.0], [0.0, 2.0]])
    np.testing.assert_array_equal(mmio.matrix_from_text(mmio.matrix_to_text(a, symmetric=False)).to_dense(),
                                  a.to_dense())
    with pytest.raises(DataFormatError):
        mmio.matrix_to_text(SparseMatrixCsr.from_dense([[1.0, 5.0], [4.0, 2.0]]), symmetric=True)


def test_comments_skipped_and_files_roundtrip(tmp_path):
    text = ("%%MatrixMarket matrix coordinate real symmetric\n% by hand\n2 2 2\n1 1 4\n% tail\n2 2 9\n")
    np.testing.assert_array_equal(mmio.matrix_from_text(text).to_dense(), np.diag([4.0, 9.0]))
    A = inputs.poisson_2d(k=8, batch=1).A
    mmio.save_matrix(tmp_path / "a.mtx", A)
    same_matrix(mmio.load_matrix(tmp_path / "a.mtx"), A)
    v = np.random.default_rng(0).standard_normal(A.n)
    mmio.save_vector(tmp_path / "b.mtx", v)
    np.testing.assert_array_equal(mmio.load_vector(tmp_path / "b.mtx"), v)


@pytest.mark.parametrize("text", [
    "2 2 1\n1 1 4\n",                                                        # no banner
    "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1\n",      # unsupported field
    "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 4\n",         # entry count
    "%%MatrixMarket matrix coordinate real general\n2 3 1\n1 1 4\n",         # not square
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 4\n",         # index range
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n",           # short entry
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 x\n",         # non-numeric
    "%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 2 4\n",       # above the diagonal
    "%%MatrixMarket matrix coordinate real general\n",                       # no size line
])
def test_malformed_matrices_raise(text):
    with pytest.raises(DataFormatError):
        mmio.matrix_from_text(text)


@pytest.mark.parametrize("text", [
    "%%MatrixMarket matrix coordinate real general\n1 1\n1\n",
    "%%MatrixMarket matrix array real general\n2 1\n1\n",
    "%%MatrixMarket matrix array real general\n1 2\n1\n",
    "%%MatrixMarket matrix array real general\n1 1\nabc\n",
])
def test_malformed_vectors_raise(text):
    with pytest.raises(DataFormatError):
        mmio.vector_from_text(text)
