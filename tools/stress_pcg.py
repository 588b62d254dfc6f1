"""Run a fixed number of PCG iterations repeatedly on the config-1 workload
and report whether the iterates are bitwise reproducible."""
import os
import sys

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
P = gnn.build_learned(model, A, rhs[:, 0])
for it in [int(x) for x in os.environ.get("ITERS", "5,20,100,400").split(",")]:
    opts = pcg.SolveOptions(thresholds=(1e-14,), max_iter=it)
    X0, _ = pcg.pcg_solve_batch(A, rhs, P, opts)
    X0 = X0.clone()
    nd = 0
    for r in range(int(os.environ.get("REPS", "6"))):
        X, _ = pcg.pcg_solve_batch(A, rhs, P, opts)
        d = X.view(torch.int64) != X0.view(torch.int64)
        if bool(d.any()):
            nd += 1
            cols = torch.nonzero(d.any(0)).flatten().tolist()
            print(f"  iters {it} rep {r}: systems differing {cols[:12]}", flush=True)
    print(f"iters {it}: {nd} runs differ", flush=True)
