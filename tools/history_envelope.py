"""Largest |log10(history / reference history)| of the device PCG on the
reference's own L' (the goldens with a recorded trace): the measured basis of
the envelope bars in tests/test_gpu_parity.py."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from golden_util import Golden

from paper_2305_16432_b200 import gnn, pcg, sparse

for name in ("cfg1_trained", "cfg1_perturbed"):
    g = Golden(name)
    c = g.case(0)
    A = sparse.SparseMatrixCsr(g.n, g.row_ptr, g.col_idx, g.values)
    P = gnn.assemble_preconditioner(c["lower"], A)
    x, rep = pcg.pcg_solve(A, g.rhs[:, 0], P, pcg.SolveOptions(thresholds=tuple(g.meta["thresholds"]),
                                                               max_iter=g.meta["max_iter"]))
    h, ref = np.array(rep.history), c["history"]
    m = min(len(h), len(ref))
    dev = np.abs(np.log10(h[:m] / ref[:m]))
    print(name, "entries", len(h), len(ref), "max deviation (decades)", float(dev.max()), "at k =", int(dev.argmax()))
