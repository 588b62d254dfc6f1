"""Per-warp timeline of the line solve (CTA 0 of the last launch), from a
library built with -DNPCG_LINE_TRACE:

    make -C paper_2305_16432_b200/csrc EXTRA=-DNPCG_LINE_TRACE OUT=../libnpcg_trace.so
    NPCG_LIB=$PWD/paper_2305_16432_b200/libnpcg_trace.so TRACE_DIR=fwd python tools/trace_line.py

TRACE_DIR=fwd runs one plain forward solve (ldlt_apply_inverse traces its
forward launch only if the backward launch is skipped: we call the raw ABI).
Prints, per warp, the first step, the clock of its first and last stage and
the mean cycles per stage (each stage = group * 4 steps).
"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2305_16432_b200 import _native, gnn, inputs, pcg
    k = int(os.environ.get("PROBE_K", "256"))
    B = int(os.environ.get("PROBE_B", "64"))
    prob = inputs.poisson_2d(k=k, batch=B)
    A = prob.A
    rng = np.random.default_rng(0)
    P = gnn.assemble_preconditioner(rng.uniform(-0.2, 0.2, A.strict_lower().nnz), A)
    rhs = torch.from_numpy(prob.rhs).cuda()
    opts = pcg.SolveOptions(thresholds=(1e-8,), max_iter=int(os.environ.get("TRACE_ITERS", "3")))
    pcg.pcg_solve_batch(A, rhs, P, opts, with_history=False)
    torch.cuda.synchronize()
    lib = _native.load_library()
    buf = (ctypes.c_longlong * (16 * 2048))()
    rc = lib.npcg_debug_line_trace(buf, 16 * 2048)
    t = np.frombuffer(buf, dtype=np.int64).reshape(16, 2048)
    t0 = min(t[w, 1] for w in range(16) if t[w, 1] > 0)
    print("rc", rc, "(last launch of the solve = backward)")
    names = ["wait", "operands", "refill", "ring in", "ring out chk", "steps", "results", "fence", "store", "loop"]
    for w in range(16):
        n = int((t[w, 1:] > 0).sum()) // 10
        if n < 3:
            continue
        ev = t[w, 1:10 * n + 1].reshape(n, 10).astype(float)
        seg = np.diff(ev, axis=1)                      # within a stage
        tail = ev[1:, 0] - ev[:-1, 9]                   # to the next stage
        per = np.median(np.diff(ev[:, 0]))
        parts = [np.median(seg[:, k]) for k in range(9)] + [np.median(tail)]
        st = np.diff(ev[:, 0])
        print(f"w{w:2d} C0={t[w,0]} start={ev[0,0]-t0:8.0f} end={ev[-1,9]-t0:8.0f} n={n} p90/stage {np.percentile(st,90):6.0f} max {st.max():6.0f} sum(wait)={seg[:,0].sum():.0f} sum(ringin)={seg[:,3].sum():.0f} sum(ringout)={seg[:,4].sum():.0f}")
        print(f"w{w:2d} cyc/stage {per:6.0f} | " + " ".join(f"{nm}={v:.0f}" for nm, v in zip(names, parts)))

if __name__ == "__main__":
    main()
