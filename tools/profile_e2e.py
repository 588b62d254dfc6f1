"""Host-side profile of the end-to-end call sequence bench.py times (config 2)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2305_16432_b200 import gnn, pcg, sparse

prob, model = bench.workload(256, 64)
A = prob.A
opts = pcg.SolveOptions(thresholds=(1e-8,))
vals_pin = torch.from_numpy(A.values.copy()).pin_memory()
rhs_pin = torch.from_numpy(prob.rhs.copy()).pin_memory()
b0_pin = torch.from_numpy(prob.rhs[:, 0].copy()).pin_memory()


def step():
    Ah = sparse.SparseMatrixCsr(A.n, A.row_ptr, A.col_idx, vals_pin.numpy())
    Ph = gnn.build_learned(model, Ah, b0_pin)
    Xh, reps = pcg.pcg_solve_batch(Ah, rhs_pin, Ph, opts)
    return Xh


for _ in range(3):
    step()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    step()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(35)
