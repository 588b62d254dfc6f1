"""One bench step (config 1) with timing and iteration counts, for debugging."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2305_16432_b200 import gnn, pcg

k = int(os.environ.get("K", "256"))
B = int(os.environ.get("B", "64"))
prob, model = bench.workload(k, B)
A = prob.A
rhs = torch.from_numpy(prob.rhs).cuda()
opts = pcg.SolveOptions(thresholds=(bench.CFG["rtol"],), max_iter=int(os.environ.get("MAXIT", "3000")))
for it in range(2):
    t0 = time.time()
    if os.environ.get("RANDOM_FACTOR"):
        rng = np.random.default_rng(0)
        P = gnn.assemble_preconditioner(rng.uniform(-0.2, 0.2, A.strict_lower().nnz), A)
    else:
        P = gnn.build_learned(model, A, rhs[:, 0])
    torch.cuda.synchronize()
    t1 = time.time()
    X, reps = pcg.pcg_solve_batch(A, rhs, P, opts, profile=True)
    torch.cuda.synchronize()
    t2 = time.time()
    its = np.array([r.iterations for r in reps])
    print(f"gnn {t1 - t0:.3f}s pcg {t2 - t1:.3f}s iters {its.min()}..{its.max()} conv {all(r.converged for r in reps)}",
          flush=True)
    p = pcg.LAST_PROFILE
    print({kk: round(p['kernel_ms'][kk] / max(p['kernel_launches'][kk], 1) * 1e3, 1) for kk in p['kernel_ms']}, flush=True)
