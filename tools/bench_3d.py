"""Configs 4 and 5 (3-D Kuhn cubes) at size on one GPU, timed like bench.py
(CUDA events, GNN and PCG apart, per-kernel-class times of a profiled solve):
config 4 -- 64^3 cells, Dirichlet eliminated, 128 RHS sharing one L';
config 5 -- 128^3 cells (2.1 M rows), distinct systems (default 8) with
their own A and L', rtol 1e-10. Prints one JSON line per config."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def model_for(gain, cfg=4):
    from paper_2305_16432_b200 import gnn
    gnn.FEATURE_WIDTH = 64
    if os.environ.get("WEIGHTS", "trained") == "trained":
        # trained on 6^3 .. 12^3 cubes by the device training step (PROBLEM=poisson3d | heat3d
        # tools/train_bench_weights.py; logs in profiles/r2_train_*3d_weights.log)
        name = "poisson3d_latent64_mp5.json" if cfg == 4 else "heat3d_latent64_mp5.json"
        return gnn.load_model(os.path.join(ROOT, "paper_2305_16432_b200", "weights", name))
    hyper = gnn.GnnHyperParams(l=1, h=64, n_mp=5, l_mp=1, h_mp=64)
    model = gnn.create_model(hyper, seed=3)
    for r in range(5):
        for s in ("node", "edge"):
            model.params[f"mp{r}.{s}.1.w"] *= gain
    return model


def run(cfg, k, batch, gain, steps):
    import torch
    import bench
    from paper_2305_16432_b200 import gnn, inputs, pcg
    t = time.time()
    prob = inputs.poisson_3d(k=k, batch=batch) if cfg == 4 else inputs.heat_3d(k=k, batch=batch)
    gen_s = time.time() - t
    A = prob.A
    model = model_for(gain, cfg)
    rhs = torch.from_numpy(prob.rhs).cuda()
    vals = torch.from_numpy(prob.values).cuda() if prob.values is not None else None
    opts = pcg.SolveOptions(thresholds=(prob.rtol,))

    def build():
        if vals is None:
            return gnn.build_learned(model, A, rhs[:, 0])
        return gnn.build_learned_batch(model, A, rhs, values=vals)

    P = build()
    if os.environ.get("PROFILE_ONLY"):  # one solve, for ncu
        opts1 = pcg.SolveOptions(thresholds=(prob.rtol,), max_iter=int(os.environ.get("PROFILE_ITERS", "3")))
        pcg.pcg_solve_batch(A, rhs, P, opts1, values=vals)
        torch.cuda.synchronize()
        return
    if os.environ.get("SWEEP"):  # "label:VAR=v,VAR=v;label:..." -> PCG time per setting
        for item in os.environ["SWEEP"].split(";"):
            label, _, kv = item.partition(":")
            for pair in filter(None, kv.split(",")):
                key, _, v = pair.partition("=")
                os.environ[key] = v
            pcg.pcg_solve_batch(A, rhs, P, opts, values=vals)
            ms = []
            for _ in range(steps):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                X, reps = pcg.pcg_solve_batch(A, rhs, P, opts, values=vals)
                e1.record()
                e1.synchronize()
                ms.append(e0.elapsed_time(e1))
            print(json.dumps({"sweep": label, "cfg": cfg, "batch": int(rhs.shape[1]), "pcg_ms": round(float(np.mean(ms)), 3),
                              "converged": bool(all(r.converged for r in reps))}), flush=True)
        return
    X, reps = pcg.pcg_solve_batch(A, rhs, P, opts, values=vals)  # warm-up
    times, g_ms, p_ms = [], [], []
    for _ in range(steps):
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        P = build()
        e[1].record()
        X, reps = pcg.pcg_solve_batch(A, rhs, P, opts, values=vals)
        e[2].record()
        e[2].synchronize()
        g_ms.append(e[0].elapsed_time(e[1]))
        p_ms.append(e[1].elapsed_time(e[2]))
        times.append(e[0].elapsed_time(e[2]))
    pcg.pcg_solve_batch(A, rhs, P, opts, values=vals, profile=True)
    prof = dict(pcg.LAST_PROFILE)
    its = np.array([r.iterations for r in reps])
    n, nnz = A.n, A.nnz
    nnzl = (nnz - n) // 2
    ML = 12 * nnzl + 4 * (n + 1)
    Bn = its.size
    distinct = vals is not None
    # bytes per kernel class (fp64 values, int32 indices)
    col_iters = int(its.sum())
    spmv_b = (col_iters * (12 * nnz + 4 * (n + 1)) if distinct else int(its.max()) * (12 * nnz + 4 * (n + 1))) + col_iters * 16 * n
    trsv_b = (col_iters * 2 * ML if distinct else int(its.max()) * 2 * ML) + col_iters * 56 * n
    km = prof["kernel_ms"]
    peak = bench.peak_hbm()
    spmv_ms = km["spmv_apdot"] + km["spmv_drift"]
    trsv_ms = km["trsv_fwd"] + km["trsv_bwd"]
    gfl = bench.gnn_flops(n, nnz, Bn if distinct else 1) / 1e9
    iter_bytes = col_iters * (12 * nnz + 4 * (n + 1) + 2 * ML + 8 * n + 104 * n) if distinct else \
        int(its.max()) * (12 * nnz + 4 * (n + 1) + 2 * ML + 8 * n) + col_iters * 104 * n
    pcg_mean = float(np.mean(p_ms))
    line = {"config": cfg, "k": k, "n": n, "nnz": nnz, "batch": Bn, "distinct_systems": distinct,
            "rtol": prob.rtol, "gain": gain, "gen_s": round(gen_s, 1),
            "weights": "trained" if os.environ.get("WEIGHTS", "trained") == "trained" else "seeded",
            "value": round(Bn / (np.mean(times) * 1e-3), 3), "unit": "systems/s", "ms_per_step": round(float(np.mean(times)), 3),
            "gnn_ms": round(float(np.mean(g_ms)), 3), "pcg_ms": round(pcg_mean, 3),
            "iterations": {"min": int(its.min()), "max": int(its.max()), "mean": float(its.mean())},
            "all_converged": bool(all(r.converged for r in reps)),
            "roofline": {"peak_gbs": peak,
                         "spmv": {"ms": round(spmv_ms, 3), "gbs": round(spmv_b / spmv_ms / 1e6, 1), "frac": round(spmv_b / spmv_ms / 1e6 / peak, 4)},
                         "sptrsv": {"ms": round(trsv_ms, 3), "gbs": round(trsv_b / trsv_ms / 1e6, 1), "frac": round(trsv_b / trsv_ms / 1e6 / peak, 4)},
                         "pcg_iteration": {"gbs": round(iter_bytes / pcg_mean / 1e6, 1), "frac": round(iter_bytes / pcg_mean / 1e6 / peak, 4)},
                         "gnn": {"gflop": round(gfl, 1), "tflops": round(gfl / float(np.mean(g_ms)), 2)}},
            "kernel_ms": {k2: round(v, 3) for k2, v in km.items()}, "passes": prof.get("passes")}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    cfg = int(os.environ.get("CFG", "4"))
    k = int(os.environ.get("K", "64" if cfg == 4 else "128"))
    batch = int(os.environ.get("BATCH", "128" if cfg == 4 else "8"))
    run(cfg, k, batch, float(os.environ.get("GAIN", "1.0")), int(os.environ.get("STEPS", "2")))
