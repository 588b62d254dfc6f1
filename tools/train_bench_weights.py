"""Train the benchmark network (latent 64, 5 rounds) with the device training
step on small Poisson problems and report what the trained L' does on
config 2 (iterations against the seeded weights, Jacobi and Gauss-Seidel).

    python tools/train_bench_weights.py            # prints progress, writes gpurun_out/poisson_f64_trained.json
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2305_16432_b200 import gnn, inputs, pcg, preconditioners, train

STEPS_EPOCHS = int(os.environ.get("EPOCHS", "6"))
LR = float(os.environ.get("LR", "1e-3"))
KS = [int(v) for v in os.environ.get("KS", "24,32,40,48").split(",")]
PER_MESH = int(os.environ.get("PER_MESH", "4"))
MESHES = int(os.environ.get("MESHES", "24"))
GAIN = float(os.environ.get("GAIN", "1.0"))
EVAL_K = int(os.environ.get("EVAL_K", "256"))
PROBLEM = os.environ.get("PROBLEM", "poisson")  # "poisson" (config 2) or "wave" (config 3: a matrix per system)
OUT = os.environ.get("OUT", "gpurun_out/poisson_f64_trained.json")
# extra tuples per mesh with a white-noise x (b = A x): ||(P - A) x||^2 over white x estimates the
# Frobenius ("naive") objective, the solution vectors alone weight the smooth modes only
NOISE = int(os.environ.get("NOISE", "0"))


def problem(k, batch, cfg):
    if PROBLEM == "wave":
        # config 3 is 512^2 cells with dt = 1e-3: the mass : dt^2-stiffness balance goes with
        # (dt / h)^2, so a k^2 training mesh gets dt scaled to keep config 3's balance
        return inputs.wave_2d(k=k, batch=batch, cfg=cfg, dt=1e-3 * 512.0 / k)
    if PROBLEM == "poisson3d":
        return inputs.poisson_3d(k=k, batch=batch, cfg=cfg)
    if PROBLEM == "heat3d":
        # config 5 is 128^3 cells with dt = 1e-3: the mass : dt-stiffness balance goes with dt / h^2,
        # so a k^3 training cube gets dt scaled to keep config 5's balance
        return inputs.heat_3d(k=k, batch=batch, cfg=cfg, dt=1e-3 * (128.0 / k) ** 2)
    return inputs.poisson_2d(k=k, batch=batch, cfg=cfg)


def system(prob, c):
    from paper_2305_16432_b200.sparse import SparseMatrixCsr
    if prob.values is None:
        return prob.A
    return SparseMatrixCsr(prob.A.n, prob.A.row_ptr, prob.A.col_idx, np.ascontiguousarray(prob.values[:, c]))


class Tup:
    def __init__(self, A, b, x):
        self.A, self.b, self.x = A, b, x


def make_tuples():
    out = []
    for j in range(MESHES):
        prob = problem(KS[j % len(KS)], PER_MESH, 50 + j)
        for c in range(PER_MESH):
            A = system(prob, c)
            x, rep = pcg.pcg_solve(A, prob.rhs[:, c].copy(), preconditioners.build_jacobi(A),
                                   pcg.SolveOptions(thresholds=(1e-12,), max_iter=20000))
            assert rep.converged
            out.append(Tup(A, prob.rhs[:, c].copy(), x))
        rng = np.random.default_rng(9000 + j)
        for c in range(NOISE):
            A = system(prob, c % PER_MESH)
            xn = rng.standard_normal(A.n) * float(np.linalg.norm(out[-1].x) / np.sqrt(A.n))
            from paper_2305_16432_b200 import sparse as _sp
            out.append(Tup(A, _sp.spmv(A, xn), xn))
    return out


def evaluate(model, tag):
    prob = problem(EVAL_K, 4 if PROBLEM in ("wave", "heat3d") else 16, {"poisson": 2, "wave": 3, "poisson3d": 4, "heat3d": 5}[PROBLEM])
    A = prob.A
    rhs = torch.from_numpy(prob.rhs).cuda()
    opts = pcg.SolveOptions(thresholds=(1e-8,), max_iter=6000)
    try:
        if prob.values is None:
            P = gnn.build_learned(model, A, rhs[:, 0])
            _, reps = pcg.pcg_solve_batch(A, rhs, P, opts)
        else:
            vals = torch.from_numpy(prob.values).cuda()
            P = gnn.build_learned_batch(model, A, rhs, values=vals)
            _, reps = pcg.pcg_solve_batch(A, rhs, P, opts, values=vals)
        its = [r.iterations for r in reps]
        print(f"[{tag}] k={EVAL_K}: iterations mean {np.mean(its):.1f} min {min(its)} max {max(its)} "
              f"converged {all(r.converged for r in reps)}", flush=True)
        return float(np.mean(its))
    except Exception as e:  # NotSpd / breakdown: report, keep going
        print(f"[{tag}] failed: {type(e).__name__}: {e}", flush=True)
        return float("inf")


def main():
    gnn.FEATURE_WIDTH = bench.CFG["width"]
    hyper = gnn.GnnHyperParams(l=1, h=bench.CFG["h"], n_mp=bench.CFG["n_mp"], l_mp=1, h_mp=bench.CFG["h"])
    model = gnn.create_model(hyper, seed=bench.CFG["seed"])
    if GAIN != 1.0:
        for r in range(hyper.n_mp):
            for s in ("node", "edge"):
                model.params[f"mp{r}.{s}.1.w"] *= GAIN
    t0 = time.time()
    tuples = make_tuples()
    print(f"{len(tuples)} tuples in {time.time() - t0:.1f}s", flush=True)
    for kind in ("jacobi", "gauss_seidel"):
        prob = problem(EVAL_K, 4, {"poisson": 2, "wave": 3, "poisson3d": 4, "heat3d": 5}[PROBLEM])
        its = []
        for c in range(4):
            A = system(prob, c)
            _, rep = pcg.pcg_solve(A, prob.rhs[:, c].copy(), preconditioners.build(kind, A),
                                   pcg.SolveOptions(thresholds=(1e-8,), max_iter=6000))
            its.append(rep.iterations)
        print(f"[{kind}] iterations mean {np.mean(its):.1f}", flush=True)
    evaluate(model, "initial")
    best = (float("inf"), None)
    for ep in range(STEPS_EPOCHS):
        cfg = train.TrainConfig(loss_kind="data", learning_rate=LR, batch_size=16, epochs=1, seed=ep)
        t0 = time.time()
        model, hist = train.train(model, tuples, cfg)
        losses = [h["batch_loss"] for h in hist]
        print(f"epoch {ep}: {len(hist)} steps in {time.time() - t0:.1f}s, batch loss {losses[0]:.4e} -> {losses[-1]:.4e} "
              f"(mean {np.mean(losses):.4e})", flush=True)
        its = evaluate(model, f"epoch {ep}")
        if its < best[0]:
            best = (its, model.copy())
    if best[1] is not None:
        os.makedirs("gpurun_out", exist_ok=True)
        gnn.save_model(OUT, best[1])
        print(json.dumps({"best_iterations_mean": best[0]}))


if __name__ == "__main__":
    main()
