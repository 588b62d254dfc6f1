"""Fixed (non-iteration) cost of one batched solve: wall time at a few
max_iter settings, extrapolated to zero iterations (for finding host-side
overhead in pcg_solve_batch)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2305_16432_b200 import gnn, pcg

prob, model = bench.workload(256, 64)
A = prob.A
rhs = torch.from_numpy(prob.rhs).cuda()
P = gnn.build_learned(model, A, rhs[:, 0])
for hist in (True, False):
    for mi in (2, 50, 200, 400):
        opts = pcg.SolveOptions(thresholds=(1e-8,), max_iter=mi)
        ts = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            X, reps = pcg.pcg_solve_batch(A, rhs, P, opts, with_history=hist)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        print(f"history={hist} max_iter={mi:4d} wall ms {1e3 * min(ts):8.2f}", flush=True)
t0 = time.perf_counter()
for _ in range(3):
    P = gnn.build_learned(model, A, rhs[:, 0])
torch.cuda.synchronize()
print(f"build_learned ms {1e3 * (time.perf_counter() - t0) / 3:8.2f}")
# a full bench step (GNN + solve to rtol), with and without the history buffer
for hist in (True, False):
    opts = pcg.SolveOptions(thresholds=(1e-8,))
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        P = gnn.build_learned(model, A, rhs[:, 0])
        X, reps = pcg.pcg_solve_batch(A, rhs, P, opts, with_history=hist)
        torch.cuda.synchronize()
        print(f"full step history={hist}: {1e3 * (time.perf_counter() - t0):8.2f} ms, "
              f"iters max {max(r.iterations for r in reps)}", flush=True)
