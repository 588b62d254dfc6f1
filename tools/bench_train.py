"""Training-step timing: one minibatch (tuple losses + gradients + Adam) on
the device against the oracle's CPU restatement of pcgkit.train on the same
tuples (config-1 shape: heat 32 x 32, HEAT_HYPER-like latent 16, 5 rounds).

    python tools/bench_train.py            # prints one JSON line
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import port, train_port
from paper_2305_16432_b200 import gnn, inputs, pcg, train

K = int(os.environ.get("K", "32"))
BATCH = int(os.environ.get("BATCH", "16"))
F = int(os.environ.get("F", "16"))
gnn.FEATURE_WIDTH = F


class Tup:
    def __init__(self, A, b, x):
        self.A, self.b, self.x = A, b, x


tuples = []
for j in range(BATCH):
    prob = inputs.heat_2d(k=K, cfg=100 + j)
    A, b = prob.A, prob.rhs[:, 0].copy()
    x, rep = pcg.pcg_solve(A, b, None, pcg.SolveOptions(thresholds=(1e-12,), max_iter=5000))
    tuples.append(Tup(A, b, x))
hyper = gnn.GnnHyperParams(l=1, h=F, n_mp=5, l_mp=1, h_mp=F)
model = gnn.create_model(hyper, seed=0)
cfg = train.TrainConfig(batch_size=BATCH)
tr = train.DeviceTrainer(model)
idx = list(range(BATCH))
for _ in range(3):
    loss, grad = train.batch_gradients(tr, tuples, idx, cfg)
torch.cuda.synchronize()
reps = 10
t0 = time.perf_counter()
for s in range(reps):
    loss, grad = train.batch_gradients(tr, tuples, idx, cfg)
    tr.adam_step(grad, s + 1, grad_scale=1.0 / BATCH)
torch.cuda.synchronize()
gpu_s = (time.perf_counter() - t0) / reps
ohp = port.Hyper(l=1, h=F, n_mp=5, l_mp=1, h_mp=F, width=F)
ot = [(port.Csr(t.A.n, t.A.row_ptr, t.A.col_idx, t.A.values), t.b, t.x) for t in tuples]
params = {k: v.copy() for k, v in model.params.items()}
t0 = time.perf_counter()
oloss, ograds = train_port.batch_gradients(ohp, params, ot, idx)
train_port.adam_step(params, ograds, {"m": {}, "v": {}}, 1)
cpu_s = time.perf_counter() - t0
print(json.dumps({"workload": f"heat {K}x{K}, latent {F}, 5 rounds, minibatch {BATCH} (loss + gradients + Adam)",
                  "n": tuples[0].A.n, "gpu_ms_per_step": round(gpu_s * 1e3, 3), "cpu_port_ms_per_step": round(cpu_s * 1e3, 1),
                  "tuples_per_s_gpu": round(BATCH / gpu_s, 1), "tuples_per_s_cpu": round(BATCH / cpu_s, 2),
                  "cpu_threads": torch.get_num_threads(), "dtype": "f64"}))
