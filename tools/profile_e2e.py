"""Wall-clock sections of the end-to-end call sequence bench.py times (config 2)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2305_16432_b200 import gnn, pcg, sparse

prob, model = bench.workload(256, 64)
A = prob.A
opts = pcg.SolveOptions(thresholds=(1e-8,))
vals_pin = torch.from_numpy(A.values.copy()).pin_memory()
rhs_pin = torch.from_numpy(prob.rhs.copy()).pin_memory()
b0_pin = torch.from_numpy(prob.rhs[:, 0].copy()).pin_memory()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
acc = {}


def tick(name, t0):
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    acc.setdefault(name, []).append((t1 - t0) * 1e3)
    return t1


for it in range(8):
    flush.fill_(1.0)
    torch.cuda.synchronize()
    t = time.perf_counter()
    t00 = t
    Ah = sparse.SparseMatrixCsr(A.n, A.row_ptr, A.col_idx, vals_pin.numpy())
    t = tick("matrix object", t)
    Ph = gnn.build_learned(model, Ah, b0_pin)
    t = tick("build_learned", t)
    Bm = sparse.to_device(rhs_pin)
    t = tick("rhs h2d", t)
    X, reps = pcg.pcg_solve_batch(Ah, Bm, Ph, opts)
    t = tick("pcg (device in/out)", t)
    Xh = sparse.to_host(X)
    t = tick("x d2h", t)
    acc.setdefault("total", []).append((t - t00) * 1e3)
    # the one-call form
    flush.fill_(1.0)
    torch.cuda.synchronize()
    t = time.perf_counter()
    Ah = sparse.SparseMatrixCsr(A.n, A.row_ptr, A.col_idx, vals_pin.numpy())
    Ph = gnn.build_learned(model, Ah, b0_pin)
    Xh, reps = pcg.pcg_solve_batch(Ah, rhs_pin, Ph, opts)
    tick("one-call total", t)
for k, v in acc.items():
    print(f"{k:24s} {np.median(v[2:]):8.3f} ms")
