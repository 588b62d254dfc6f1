"""Config 4 (BASELINE.json): 3-D Poisson on a jittered 64^3 Kuhn cube
(n = 250,047 free), batch of GRF right-hand sides, one shared L' from the
GNN (reference-mode architecture, latent 64, 5 rounds), PCG rtol 1e-8. The
3-D pattern runs the level-set triangular solves. One JSON line:
systems/s (GNN + batched PCG per step, CUDA events) and the per-iteration
HBM figure of SURVEY.md 8(d) (M + B V).

    python tools/bench_cfg4.py [--k 64] [--batch 128] [--steps 2]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2305_16432_b200 import gnn, inputs, pcg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=int, default=64)
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--max-iter", type=int, default=3000)
    ap.add_argument("--gain", type=float, default=1.0,
                    help="processor output-layer gain (bench.py's 2-D workload uses 10; at 3-D that factor diverges)")
    a = ap.parse_args()
    t0 = time.time()
    prob = inputs.poisson_3d(k=a.k, batch=a.batch)
    t_gen = time.time() - t0
    A = prob.A
    gnn.FEATURE_WIDTH = bench.CFG["width"]
    hyper = gnn.GnnHyperParams(l=1, h=bench.CFG["h"], n_mp=bench.CFG["n_mp"], l_mp=1, h_mp=bench.CFG["h"])
    model = gnn.create_model(hyper, seed=bench.CFG["seed"])
    for r in range(hyper.n_mp):
        for s in ("node", "edge"):
            model.params[f"mp{r}.{s}.1.w"] *= a.gain
    rhs = torch.from_numpy(prob.rhs).cuda()
    opts = pcg.SolveOptions(thresholds=(1e-8,), max_iter=a.max_iter)

    def step(profile=False):
        P = gnn.build_learned(model, A, rhs[:, 0])
        return pcg.pcg_solve_batch(A, rhs, P, opts, with_history=False, profile=profile)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    times = []
    for _ in range(a.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        X, reps = step()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = float(np.median(times))
    its = np.array([r.iterations for r in reps])
    step(profile=True)
    prof = dict(pcg.LAST_PROFILE)
    nL = A.strict_lower().nnz
    n = A.n
    ML = 12 * nL + 4 * (n + 1)
    M = 12 * A.nnz + 4 * (n + 1) + 2 * ML + 8 * n
    iter_bytes = int(its.max()) * M + int(its.sum()) * 104 * n
    gbs = iter_bytes / (ms * 1e-3) / 1e9
    print(json.dumps({
        "metric": "systems solved to rtol 1e-8 /sec (config 4)", "value": round(a.batch / (ms * 1e-3), 3),
        "unit": "systems/s", "ms_per_step": round(ms, 3), "steps": a.steps,
        "config": {"workload": f"cfg4 poisson-3d {a.k}^3 Kuhn cube jittered 0.15h, Dirichlet-eliminated "
                               f"(n={n}, nnz={A.nnz}), {a.batch} GRF RHS, one shared L' (latent 64, 5 rounds, "
                               f"create_model(seed={bench.CFG['seed']}), processor output gain x{a.gain:g})",
                   "host_generation_s": round(t_gen, 1)},
        "iterations": {"min": int(its.min()), "max": int(its.max()), "mean": float(its.mean())},
        "all_converged": bool(all(r.converged for r in reps)),
        "pcg_iteration_roofline": {"achieved_gbs": round(gbs, 1), "bytes_per_iter_at_B": int(M + a.batch * 104 * n),
                                   "frac_of_measured": round(gbs / bench.peak_hbm(), 4)},
        "kernel_ms": {k: round(v, 3) for k, v in prof.get("kernel_ms", {}).items()},
        "streams": prof.get("streams", 1)}))


if __name__ == "__main__":
    main()
