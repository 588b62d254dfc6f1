"""Repeat the batched triangular solves (P^{-1} r, 64 right-hand sides) on
the config-1 pattern and check the results are bitwise stable."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2305_16432_b200 import gnn, inputs, sparse

k = int(os.environ.get("K", "256"))
B = int(os.environ.get("B", "64"))
reps = int(os.environ.get("REPS", "50"))
prob = inputs.poisson_2d(k=k, batch=B)
A = prob.A
rng = np.random.default_rng(0)
P = gnn.assemble_preconditioner(rng.uniform(-0.2, 0.2, A.strict_lower().nnz), A)
pat, S, D = P.factor.device()
r = torch.from_numpy(prob.rhs).cuda().contiguous()
z0 = sparse.apply_inverse_device(pat, S, False, D, False, r, B)
torch.cuda.synchronize()
bad = 0
for i in range(reps):
    z = sparse.apply_inverse_device(pat, S, False, D, False, r, B)
    d = (z.view(torch.int64) != z0.view(torch.int64))
    if bool(d.any()):
        bad += 1
        rows, cols = torch.nonzero(d, as_tuple=True)
        print(f"rep {i}: {int(d.sum())} mismatches, systems {sorted(set(cols.tolist()))[:10]}, "
              f"rows {rows.min().item()}..{rows.max().item()}", flush=True)
print(f"{bad} of {reps} repetitions differ")
