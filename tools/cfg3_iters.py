"""Iteration counts of config 3's systems (wave 512^2, 32 distinct systems)
for seeded latent-64 weights at several processor-output gains, and for
Jacobi, on the device."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2305_16432_b200 import gnn, inputs, pcg, preconditioners
    prob = inputs.wave_2d(k=int(os.environ.get("K", "512")), batch=32)
    A, vals = prob.A, torch.from_numpy(prob.values).cuda()
    rhs = torch.from_numpy(prob.rhs).cuda()
    gnn.FEATURE_WIDTH = 64
    opts = pcg.SolveOptions(thresholds=(1e-8,))
    for gain in (10.0, 5.0, 3.0, 2.0, 1.0):
        hyper = gnn.GnnHyperParams(l=1, h=64, n_mp=5, l_mp=1, h_mp=64)
        model = gnn.create_model(hyper, seed=3)
        for r in range(5):
            for s in ("node", "edge"):
                model.params[f"mp{r}.{s}.1.w"] *= gain
        P = gnn.build_learned_batch(model, A, rhs, values=vals)
        X, reps = pcg.pcg_solve_batch(A, rhs, P, opts, values=vals, with_history=False)
        its = np.array([r.iterations for r in reps])
        print(f"gain {gain}: mean {its.mean():.1f} max {its.max()} min {its.min()} conv {all(r.converged for r in reps)} "
              f"|L'|max {float(P.device_factor()[1].abs().max()):.3f}", flush=True)
    # Jacobi: the same device path with L' = 0
    Dv = torch.empty((A.n, 32), dtype=torch.float64, device="cuda")
    its = []
    for j in range(32):
        Aj = A.with_values(prob.values[:, j].copy())
        J = preconditioners.build_jacobi(Aj)
        x, rep = pcg.pcg_solve(Aj, prob.rhs[:, j], J, opts)
        its.append(rep.iterations)
    print("jacobi:", np.mean(its), max(its), min(its))


if __name__ == "__main__":
    main()
