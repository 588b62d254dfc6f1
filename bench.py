#!/usr/bin/env python
"""bench.py -- NeuralPCG solve path on B200 (BASELINE.json headline metric).

Workload (config 2 of BASELINE.json, the config the metric is quoted on):
2-D Poisson, 256 x 256 jittered triangulated unit square, full-boundary
Dirichlet eliminated (n = 65,025, nnz = 453,137), 64 right-hand sides
(GRF loads), ONE shared learned factor L' from the GNN (reference-mode
architecture at latent 64, 5 message-passing rounds, seeded weights with
the processor output gain cancelled) computed on RHS 0, PCG to rtol 1e-8.

A step = build_learned (GNN on the device) + one batched PCG over the 64
right-hand sides; a unit = one right-hand side solved to rtol; metric =
units / second (whole job, all ranks). ``value`` has inputs resident in HBM;
``e2e`` runs the same step through the public API from pinned host buffers
with the host<->device copies inside the timed region. L2 is flushed
(256 MiB write) before every timed step, outside the timed interval.

Multi-GPU: one process per GPU (torchrun), each rank solves its own batch
of 64 right-hand sides on the shared mesh (weak scaling, no collective in
the data path; barrier + max-over-ranks timing only).

``--impl reference`` times the reference's CPU implementation of the same
path on the host cores (the oracle port, oracle/port.py: the reference has
no compiled artefact to build), see reference_arm().
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG = dict(k=256, jitter=0.2, batch=64, rtol=1e-8, width=64, h=64, n_mp=5, seed=3)
METRIC = "systems solved to rtol 1e-8 /sec; PCG-iteration HBM GB/s vs 8 TB/s peak"
UNIT = "systems/s"


def args_():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--k", type=int, default=CFG["k"], help="mesh cells per side (256 = config 2)")
    ap.add_argument("--batch", type=int, default=CFG["batch"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile-only", action="store_true", help="one profiled step, no JSON (for ncu)")
    return ap.parse_args()


def workload(k, batch, rank=0):
    from paper_2305_16432_b200 import gnn, inputs
    prob = inputs.poisson_2d(k=k, batch=batch, first=rank * batch)
    gnn.FEATURE_WIDTH = CFG["width"]
    hyper = gnn.GnnHyperParams(l=1, h=CFG["h"], n_mp=CFG["n_mp"], l_mp=1, h_mp=CFG["h"])
    model = gnn.create_model(hyper, seed=CFG["seed"])
    for r in range(hyper.n_mp):  # cancel the 0.1 init gain: a non-trivial L'
        for s in ("node", "edge"):
            model.params[f"mp{r}.{s}.1.w"] *= 10.0
    return prob, model


def config_dict(prob, k, batch, world):
    A = prob.A
    return {
        "workload": f"cfg2 poisson-2d {k}x{k} jittered P1, Dirichlet-eliminated (n={A.n}, nnz={A.nnz}), "
                    f"{batch} GRF right-hand sides per GPU, one shared L' from the GNN "
                    f"(latent {CFG['width']}, {CFG['n_mp']} rounds) per step, PCG rtol {CFG['rtol']}",
        "n": A.n, "nnz": A.nnz, "rhs_per_gpu": batch, "gnn": f"reference-mode F={CFG['width']} h={CFG['h']} "
        f"n_mp={CFG['n_mp']}, create_model(seed={CFG['seed']}) with processor output layers x10",
        "l2": "flushed (256 MiB write) before every timed step",
        "parallelism": f"batch-parallel x{world} (weak)",
    }


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md recipe)
# ---------------------------------------------------------------------------

REASONS = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]


class ClockSampler:
    def __init__(self, index):
        q = "clocks.sm,clocks.max.sm," + ",".join(f"clocks_event_reasons.{r}" for r in REASONS)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, mx, seen = [], [], set()
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 2 + len(REASONS):
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for r, v in zip(REASONS, f[2:]):
                if v.lower().startswith("active"):
                    seen.add(r)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(seen), "samples": len(sm)}


# ---------------------------------------------------------------------------
# roofline bookkeeping
# ---------------------------------------------------------------------------


def roofline(A, nnz_lower, prof, iters, peak_gbs, step_ms=None):
    """Achieved algorithmic GB/s of the dominant kernel (ldlt_line_kernel:
    forward solve, y / D and backward solve in one launch) and of a whole PCG
    iteration.

    Per launch, fp64 values / int32 indices, compulsory traffic only:
      factor of both directions 2 (12 nnz(L) + 4(n+1)) + D and 1/D 16 n
      + per solving column 56 n (forward: read r, Ap, write r_{k+1}, y;
        backward: read y, r, write z).
    Whole iteration: M + B V with
      M = 12 nnz(A) + 4(n+1) + 2 (12 nnz(L) + 4(n+1)) + 8 n,  V = 104 n.
    """
    n, nnz = A.n, A.nnz
    ML = 12 * nnz_lower + 4 * (n + 1)
    col_iters = int(np.sum(iters))
    nl = prof["kernel_launches"]["trsv_fwd"] + prof["kernel_launches"]["trsv_bwd"]
    ncol = len(iters)
    solves = col_iters + ncol  # every iteration plus the initial z = P^-1 r
    trsv_bytes = nl * (2 * ML + 16 * n) + solves * 56 * n
    t_trsv = (prof["kernel_ms"]["trsv_fwd"] + prof["kernel_ms"]["trsv_bwd"]) * 1e-3
    achieved = trsv_bytes / t_trsv / 1e9
    M = 12 * nnz + 4 * (n + 1) + 2 * ML + 8 * n
    iter_bytes = int(np.max(iters)) * M + col_iters * 104 * n
    # the batch runs as concurrent sub-batches (pcg.SPLIT_STREAMS): summed
    # kernel time overstates the loop, the timed step (GNN included) does not
    t_loop = sum(prof["kernel_ms"].values()) * 1e-3
    t_iter = step_ms * 1e-3 if step_ms else t_loop
    iter_gbs = iter_bytes / t_iter / 1e9
    return {
        "kernel": "ldlt_line_kernel (forward solve + y/D + backward solve, one launch per pass)",
        "bound": "hbm", "achieved": round(achieved, 1), "peak": peak_gbs, "unit": "GB/s",
        "frac": round(achieved / peak_gbs, 4), "peak_source": "measured (MEASURED_PEAKS.json hbm_gbs)",
        "traffic": ncu_traffic(),
        "launch_ms": round(t_trsv * 1e3 / max(nl, 1), 4),
        "bytes_per_launch": int(trsv_bytes / max(nl, 1)),
        "pcg_iteration": {"achieved": round(iter_gbs, 1), "frac_of_measured": round(iter_gbs / peak_gbs, 4),
                          "frac_of_8TBs": round(iter_gbs / 8000.0, 4), "bytes": int(iter_bytes),
                          "time_ms": round(t_iter * 1e3, 3),
                          "time_from": "timed step (GNN + whole batched solve)" if step_ms else "summed kernel time",
                          "summed_kernel_ms": round(t_loop * 1e3, 3), "streams": prof.get("streams", 1)},
        "kernel_ms": {k: round(v, 3) for k, v in prof["kernel_ms"].items()},
        "kernel_share": {k: round(v / max(sum(prof["kernel_ms"].values()), 1e-9), 4)
                         for k, v in prof["kernel_ms"].items()},
    }


def ncu_traffic():
    """dram bytes per trsv launch from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "trsv_ncu_summary.json")
    try:
        with open(path) as fh:
            return json.load(fh).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        return 6650.0  # B200_PROFILING.md fallback


# ---------------------------------------------------------------------------
# CPU side: the oracle port of the reference path on the host cores
# ---------------------------------------------------------------------------

_CPU = {}


def _cpu_worker_init():
    # one BLAS thread per worker process: the reference solve is sequential and
    # the parent's BLAS pool (already loaded) would otherwise oversubscribe
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)


def _cpu_solve(j):
    from oracle import port
    A, F, rhs = _CPU["A"], _CPU["F"], _CPU["rhs"]
    t = time.perf_counter()
    x, rep = port.pcg_solve(A, rhs[:, j], F, thresholds=(CFG["rtol"],))
    return time.perf_counter() - t, rep.iterations, rep.converged


def cpu_reference(prob, model, steps, warmup, cores=None):
    """Reference path (oracle port of pcgkit: numpy GNN + sequential C
    SpMV / SpTRSV, fp64) on the host: the GNN once with all BLAS threads,
    then rounds of `cores` right-hand sides in parallel (one process per
    core, single-threaded each -- the reference solve is sequential).
    Step time = t_gnn + ceil(B / cores) * t_round, i.e. the full 64-RHS step
    extrapolated from the measured round. Returns (value, info)."""
    import multiprocessing as mp
    from oracle import port
    cores = cores or len(os.sched_getaffinity(0))
    A = port.Csr(prob.A.n, prob.A.row_ptr, prob.A.col_idx, prob.A.values)
    hp = port.Hyper(l=1, h=CFG["h"], n_mp=CFG["n_mp"], l_mp=1, h_mp=CFG["h"], width=CFG["width"])
    t = time.perf_counter()
    F = port.build_learned(hp, model.params, A, prob.rhs[:, 0])
    t_gnn = time.perf_counter() - t
    _CPU.update(A=A, F=F, rhs=prob.rhs)
    B = prob.rhs.shape[1]
    per_round = min(cores, B)
    ctx = mp.get_context("fork")
    rounds = []
    its = []
    with ctx.Pool(per_round, initializer=_cpu_worker_init) as pool:
        for s in range(warmup + steps):
            cols = [(s * per_round + j) % B for j in range(per_round)]
            t = time.perf_counter()
            res = pool.map(_cpu_solve, cols)
            dt = time.perf_counter() - t
            if s >= warmup:
                rounds.append(dt)
                its.extend(r[1] for r in res)
    step_s = [t_gnn + math.ceil(B / per_round) * r for r in rounds]
    value = B / statistics.mean(step_s)
    info = {"t_gnn_s": round(t_gnn, 3), "t_round_s": round(statistics.mean(rounds), 3),
            "rhs_per_round": per_round, "iterations_mean": float(np.mean(its)) if its else None}
    return value, cores, step_s, info


def reference_arm(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    prob, model = workload(a.k, a.batch)
    value, cores, step_s, info = cpu_reference(prob, model, a.steps, a.warmup)
    sample = (f"oracle port of the reference (numpy GNN + sequential C kernels, fp64): GNN once "
              f"({info['t_gnn_s']} s, all BLAS threads) + {a.steps} timed rounds of {info['rhs_per_round']} "
              f"RHS solved in parallel (1 process/core); step = GNN + ceil({a.batch}/{info['rhs_per_round']}) rounds")
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
            "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": round(statistics.mean(step_s) * 1e3, 1), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(prob, a.k, a.batch, 1),
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": sample, **info},
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------


def main():
    a = args_()
    if a.impl == "reference":
        return reference_arm(a)
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)

    from paper_2305_16432_b200 import _native, gnn, pcg, sparse
    prob, model = workload(a.k, a.batch, rank)
    A = prob.A
    B = a.batch
    opts = pcg.SolveOptions(thresholds=(CFG["rtol"],))
    rhs_dev = torch.from_numpy(prob.rhs).cuda()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MiB

    def step(profile=False):
        P = gnn.build_learned(model, A, rhs_dev[:, 0])
        X, reps = pcg.pcg_solve_batch(A, rhs_dev, P, opts, profile=profile)
        return X, reps

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    if a.profile_only:
        step()
        torch.cuda.synchronize()
        return 0

    for _ in range(a.warmup):
        step()
    barrier()
    lib = _native.lib()
    launches0 = lib.npcg_launch_count()
    clocks = ClockSampler(local) if rank == 0 else None
    times, reps_all = [], None
    for _ in range(a.steps):
        flush.fill_(1.0)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        X, reps = step()
        e1.record()
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
        reps_all = reps
    barrier()
    clk = clocks.stop() if clocks else None
    launches = lib.npcg_launch_count() - launches0
    ms = max_over_ranks(statistics.mean(times))
    value = B * world / (ms * 1e-3)
    iters = np.array([r.iterations for r in reps_all])
    converged = all(r.converged for r in reps_all)

    # roofline: one profiled step (per-launch CUDA events, same stream)
    flush.fill_(1.0)
    barrier()
    P = gnn.build_learned(model, A, rhs_dev[:, 0])
    pcg.pcg_solve_batch(A, rhs_dev, P, opts, profile=True)
    prof = dict(pcg.LAST_PROFILE)
    nnz_lower = (A.nnz - A.n) // 2
    roof = roofline(A, nnz_lower, prof, prof["iterations"], peak_hbm(), step_ms=ms)

    # e2e through the public API from pinned host buffers
    e2e = None
    if not a.no_e2e:
        vals_pin = torch.from_numpy(A.values.copy()).pin_memory()
        rhs_pin = torch.from_numpy(prob.rhs.copy()).pin_memory()
        b0_pin = torch.from_numpy(prob.rhs[:, 0].copy()).pin_memory()
        e2e_t = []
        for s in range(a.warmup + a.steps):
            flush.fill_(1.0)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            Ah = sparse.SparseMatrixCsr(A.n, A.row_ptr, A.col_idx, vals_pin.numpy())
            Ph = gnn.build_learned(model, Ah, b0_pin)
            Xh, reps_h = pcg.pcg_solve_batch(Ah, rhs_pin, Ph, opts)  # host in -> host out
            e1.record()
            e1.synchronize()
            if s >= a.warmup:
                e2e_t.append(e0.elapsed_time(e1))
        e2e_ms = max_over_ranks(statistics.mean(e2e_t))
        e2e = {"value": round(B * world / (e2e_ms * 1e-3), 3), "unit": UNIT,
               "h2d_bytes_per_step": int(A.nnz * 8 + A.n * B * 8 + A.n * 8),
               "d2h_bytes_per_step": int(A.n * B * 8 + B * (int(iters.max()) + 1) * 8),
               "ms_per_step": round(e2e_ms, 3)}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        v, cores, step_s, info = cpu_reference(prob, model, steps=1, warmup=0)
        cpu = {"value": round(v, 4), "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"GNN once + one round of {info['rhs_per_round']} RHS on {cores} cores, "
                         f"step extrapolated to {B} RHS", **info}
    total_launches = int(sum_over_ranks(launches))
    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
                "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded jittered mesh + GRF loads; seeded GNN weights)",
                "config": config_dict(prob, a.k, B, world), "roofline": roof, "cpu_baseline": cpu,
                "e2e": e2e, "gpu_launches": total_launches, "clocks": clk,
                "iterations": {"min": int(iters.min()), "max": int(iters.max()), "mean": float(iters.mean())},
                "all_converged": converged, "gnn_dtype": "f32", "pcg_dtype": "f64"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
