"""Mint the Matrix Market goldens with the reference's own writer
(pcgkit.mmio, run in the build container where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_mmio_golden.py

The matrix is config 1's heat matrix at k = 4 (inputs.heat_2d), the vector
its right-hand side plus a few awkward values."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from pcgkit import mmio as ref_mmio  # noqa: E402
from pcgkit.sparse import SparseMatrixCsr as RefCsr  # noqa: E402

from paper_2305_16432_b200 import inputs  # noqa: E402

p = inputs.heat_2d(k=4)
A = RefCsr(p.A.n, p.A.row_ptr.copy(), p.A.col_idx.copy(), p.A.values.copy())
v = np.concatenate([p.rhs[:, 0], [1.0 / 3.0, -2.5e-308, 0.0, -0.0, 1e300]])
with open(os.path.join(HERE, "mmio_heat4_symmetric.mtx"), "w") as fh:
    fh.write(ref_mmio.matrix_to_text(A, symmetric=True))
with open(os.path.join(HERE, "mmio_heat4_general.mtx"), "w") as fh:
    fh.write(ref_mmio.matrix_to_text(A, symmetric=False))
with open(os.path.join(HERE, "mmio_heat4_rhs.mtx"), "w") as fh:
    fh.write(ref_mmio.vector_to_text(v))
print("wrote", A.n, len(v))
