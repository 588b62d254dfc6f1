"""Wall time of repeated full solves in one process; the profiled ones dump
per-launch times so a slow solve can be compared kernel by kernel."""
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2305_16432_b200 import _native, gnn, pcg

prob, model = bench.workload(256, 64)
A = prob.A
rhs = torch.from_numpy(prob.rhs).cuda()
opts = pcg.SolveOptions(thresholds=(1e-8,))
NAMES = ["spmv_apdot", "trsv_fwd", "spmv_drift", "trsv_bwd", "pupd", "other"]
lib = _native.lib()
for it in range(8):
    prof = it % 2 == 1
    if prof:
        path = tempfile.mktemp(suffix=".txt")
        os.environ["NPCG_PROFILE_DUMP"] = path
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    P = gnn.build_learned(model, A, rhs[:, 0])
    X, reps = pcg.pcg_solve_batch(A, rhs, P, opts, profile=prof)
    torch.cuda.synchronize()
    wall = 1e3 * (time.perf_counter() - t0)
    msg = f"solve {it} profile={prof} wall {wall:8.1f} ms"
    if prof:
        del os.environ["NPCG_PROFILE_DUMP"]
        d = np.loadtxt(path, ndmin=2)
        os.unlink(path)
        tot = d[:, 1].sum()
        per = {NAMES[s]: round(float(np.median(d[d[:, 0] == s, 1])) * 1e3, 1) for s in range(5) if (d[:, 0] == s).any()}
        mx = {NAMES[s]: round(float(np.max(d[d[:, 0] == s, 1])) * 1e3, 1) for s in range(5) if (d[:, 0] == s).any()}
        msg += f" kernels {tot:8.1f} ms median us {per} max us {mx}"
    print(msg, flush=True)
