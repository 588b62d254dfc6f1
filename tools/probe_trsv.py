"""Sweep the triangular-solve schedule knobs on the config-2 workload and
print the average launch time per kernel class (profiled PCG, 30 passes).

    python tools/probe_trsv.py            # one subprocess per setting
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def one():
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    from paper_2305_16432_b200 import gnn, inputs, pcg
    k = int(os.environ.get("PROBE_K", "256"))
    B = int(os.environ.get("PROBE_B", "64"))
    prob = inputs.poisson_2d(k=k, batch=B)
    A = prob.A
    low = A.strict_lower()
    rng = np.random.default_rng(0)
    P = gnn.assemble_preconditioner(rng.uniform(-0.2, 0.2, low.nnz), A)
    rhs = torch.from_numpy(prob.rhs).cuda()
    opts = pcg.SolveOptions(thresholds=(1e-8,), max_iter=30)
    pcg.pcg_solve_batch(A, rhs, P, opts, with_history=False)
    pcg.pcg_solve_batch(A, rhs, P, opts, with_history=False, profile=True)
    p = pcg.LAST_PROFILE
    ms, nl = p["kernel_ms"], p["kernel_launches"]
    print(json.dumps({k: round(ms[k] / max(nl[k], 1) * 1e3, 1) for k in ms if nl[k]}))


def sweep(settings):
    for s in settings:
        env = dict(os.environ, **s)
        r = subprocess.run([sys.executable, __file__, "one"], env=env, capture_output=True, text=True, timeout=300)
        print(s, (r.stdout.strip() or r.stderr.strip()[-400:]), flush=True)


DEFAULT = [dict(NPCG_GROUP=str(g), NPCG_CHUNK_ROWS=str(r), NPCG_PREFETCH=str(pd), NPCG_SMEM_KB="200")
           for g in (1,) for r in (65025, 32513, 16257, 8129) for pd in (4, 8)]

if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "one":
        one()
    else:
        sweep(json.loads(sys.argv[1]) if len(sys.argv) > 1 else DEFAULT)
