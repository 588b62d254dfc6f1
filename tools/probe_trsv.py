"""Per-launch kernel times of the config-1 PCG loop (profiled, 30
iterations): median over the launches that did work (the pass budget adds
cheap all-skip launches at the end, which a plain mean would average in).

    python tools/probe_trsv.py one          # this process
    python tools/probe_trsv.py '[{...}]'    # one subprocess per env setting
"""
import json
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NAMES = ["spmv_apdot", "trsv_fwd", "spmv_drift", "trsv_bwd", "pupd", "other"]


def one():
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    from paper_2305_16432_b200 import gnn, inputs, pcg
    k = int(os.environ.get("PROBE_K", "256"))
    B = int(os.environ.get("PROBE_B", "64"))
    its = int(os.environ.get("PROBE_ITERS", "30"))
    prob = inputs.poisson_2d(k=k, batch=B)
    A = prob.A
    rng = np.random.default_rng(0)
    P = gnn.assemble_preconditioner(rng.uniform(-0.2, 0.2, A.strict_lower().nnz), A)
    rhs = torch.from_numpy(prob.rhs).cuda()
    opts = pcg.SolveOptions(thresholds=(1e-14,), max_iter=its)
    pcg.pcg_solve_batch(A, rhs, P, opts, with_history=False)  # warm-up
    with tempfile.NamedTemporaryFile(suffix=".txt", delete=False) as f:
        path = f.name
    os.environ["NPCG_PROFILE_DUMP"] = path
    pcg.pcg_solve_batch(A, rhs, P, opts, with_history=False, profile=True)
    del os.environ["NPCG_PROFILE_DUMP"]
    d = np.loadtxt(path, ndmin=2)
    os.unlink(path)
    out = {}
    for slot, name in enumerate(NAMES):
        t = d[d[:, 0] == slot, 1] * 1e3
        if len(t):
            t = t[t > 0.3 * t.max()]  # launches that did work
            out[name] = round(float(np.median(t)), 1)
    print(json.dumps(out))


def sweep(settings):
    for s in settings:
        env = dict(os.environ, **s)
        r = subprocess.run([sys.executable, __file__, "one"], env=env, capture_output=True, text=True, timeout=300)
        print(s, (r.stdout.strip() or r.stderr.strip()[-400:]), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "one":
        one()
    else:
        sweep(json.loads(sys.argv[1]) if len(sys.argv) > 1 else [{}])
