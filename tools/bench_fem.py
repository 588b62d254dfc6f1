"""Device P1 assembly (csrc/fem.cu) at config 3's size: 512 x 512 jittered
square (263,169 vertices, 1,838,081 nnz), B systems with their own per-element
coefficient c = exp(0.5 GRF), A_b = M + dt^2 K_{c_b} (inputs.wave_2d), one
JSON line. The CPU column is the numpy host assembly of the same matrices
(inputs.Assembler: fem.py's element blocks + lexsort/reduceat scatter) on the
host cores, timed on a bounded sample of systems.

    python tools/bench_fem.py [--k 512] [--batch 32] [--steps 10]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2305_16432_b200 import _native, inputs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=int, default=512)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--cpu-systems", type=int, default=2)
    a = ap.parse_args()
    rng = np.random.default_rng(np.random.SeedSequence(3017).entropy)
    mesh = inputs.unit_square(a.k, 0.2, rng)
    nt, nv = len(mesh.triangles), len(mesh.vertices)
    cent = mesh.vertices[mesh.triangles].mean(axis=1)
    C = np.stack([np.exp(0.5 * inputs.grf_2d(cent, r, r.uniform(0.05, 0.3))) for r in inputs.streams(3, a.batch)],
                 axis=1)
    dt2 = 1e-3 * 1e-3
    dev = inputs.DeviceAssembler(nv, mesh.triangles)
    V = torch.from_numpy(mesh.vertices).cuda()
    Cd = torch.from_numpy(C).cuda()
    out = dev.values(V, coef=Cd, mode="M+sK", scale=dt2)  # warm + validation
    lib = _native.lib()
    for _ in range(a.warmup):
        dev.values(V, coef=Cd, mode="M+sK", scale=dt2, check=False)
    torch.cuda.synchronize()
    l0 = lib.npcg_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        dev.values(V, coef=Cd, mode="M+sK", scale=dt2, check=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    launches = (lib.npcg_launch_count() - l0) / a.steps
    # bitwise spot check of two systems against the host assembly (and its timing)
    K, M = inputs.element_blocks(mesh)
    asm = inputs.Assembler(nv, mesh.triangles)
    t0 = time.perf_counter()
    Mv = asm.values(M)
    host = []
    a.cpu_systems = min(a.cpu_systems, a.batch)
    for b in range(a.cpu_systems):
        host.append(Mv + dt2 * asm.values(K * C[:, b, None, None]))
    t_cpu = (time.perf_counter() - t0) / a.cpu_systems
    got = out[:, :a.cpu_systems].cpu().numpy()
    bitwise = bool(np.array_equal(got.view(np.int64), np.stack(host, axis=1).view(np.int64)))
    nnz = dev.nnz
    algo = nnz * a.batch * 8 + nt * a.batch * 8 + 9 * nt * 4 + (nnz + 1) * 4 + 12 * nt + 16 * nv
    peak = 6441.6
    try:
        peak = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                  "MEASURED_PEAKS.json")))["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        pass
    gbs = algo / (ms * 1e-3) / 1e9
    print(json.dumps({
        "metric": "systems assembled /sec (P1, A = M + dt^2 K_c, per-system element coefficients)",
        "value": round(a.batch / (ms * 1e-3), 1), "unit": "systems/s", "ms_per_call": round(ms, 4),
        "config": {"workload": f"cfg3 mesh {a.k}x{a.k} jittered (nv={nv}, nt={nt}, nnz={nnz}), B={a.batch}"},
        "gpu_launches_per_call": launches,
        "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(gbs / peak, 4), "bytes_per_call": int(algo)},
        "cpu_baseline": {"value": round(1.0 / t_cpu, 3), "unit": "systems/s", "cores": 1, "kind": "port",
                         "sample": f"{a.cpu_systems} systems through inputs.Assembler (numpy, fem.py order)"},
        "bitwise_vs_host": bitwise}))


if __name__ == "__main__":
    main()
