"""Per-level latency of the triangular-solve machinery: a tridiagonal SPD
matrix is a pure dependency chain (one row per level), so the profiled
forward / backward launch time divided by n is the cost of one level step.

    NPCG_CHUNK_ROWS=<n> python tools/probe_chain.py [n] [B]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2305_16432_b200 import gnn, pcg, sparse  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
i = np.arange(n)
rows = np.concatenate([i, i[1:], i[:-1]])
cols = np.concatenate([i, i[:-1], i[1:]])
vals = np.concatenate([np.full(n, 4.0), np.full(n - 1, -1.0), np.full(n - 1, -1.0)])
A = sparse.SparseMatrixCsr.from_coo(n, rows, cols, vals)
P = gnn.assemble_preconditioner(np.full(n - 1, -0.25), A)
rhs = torch.from_numpy(np.random.default_rng(0).standard_normal((n, B))).cuda()
opts = pcg.SolveOptions(thresholds=(1e-8,), max_iter=6)
pcg.pcg_solve_batch(A, rhs, P, opts, with_history=False)
pcg.pcg_solve_batch(A, rhs, P, opts, with_history=False, profile=True)
p = pcg.LAST_PROFILE
ms, nl = p["kernel_ms"], p["kernel_launches"]
print(json.dumps({k: round(ms[k] / max(nl[k], 1) * 1e6 / n, 1) for k in ("trsv_fwd", "trsv_bwd")}), "ns/level")
