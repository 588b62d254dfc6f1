"""Per-step wall times of the default bench step (device-resident inputs) over many steps:
where do the slow outliers come from (GNN call, PCG call, Python GC)?"""
import gc
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
opts = pcg.SolveOptions(thresholds=(1e-8,))
rhs = torch.from_numpy(prob.rhs).cuda()
N = int(os.environ.get("N", "300"))
for mode in ("gc on", "gc off"):
    if mode == "gc off":
        gc.collect()
        gc.disable()
    tg, tp = [], []
    for i in range(N):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        P = gnn.build_learned(model, A, rhs[:, 0])
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        X, reps = pcg.pcg_solve_batch(A, rhs, P, opts)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        tg.append((t1 - t0) * 1e3)
        tp.append((t2 - t1) * 1e3)
    tg, tp = np.array(tg[5:]), np.array(tp[5:])
    tot = tg + tp
    print(f"[{mode}] step mean {tot.mean():.2f} median {np.median(tot):.2f} p99 {np.percentile(tot, 99):.2f} max {tot.max():.2f} | "
          f"gnn median {np.median(tg):.2f} max {tg.max():.2f} | pcg median {np.median(tp):.2f} max {tp.max():.2f} | "
          f"steps > 1.2 x median: {(tot > 1.2 * np.median(tot)).sum()} of {len(tot)}", flush=True)
    slow = np.flatnonzero(tot > 1.2 * np.median(tot))
    print("   slow steps at", slow[:20].tolist(), "gnn", np.round(tg[slow][:10], 1).tolist(), "pcg", np.round(tp[slow][:10], 1).tolist())
