"""Timeline of the warp-specialised line P^{-1} (ldlt_line_kernel) for CTA 0
of system 0 of the last launch, from a library built with -DNPCG_LINE_TRACE:

    make -C paper_2305_16432_b200/csrc EXTRA=-DNPCG_LINE_TRACE \
        OUT=../libnpcg_trace.so OBJDIR=../../build/obj_trace
    NPCG_LIB=$PWD/paper_2305_16432_b200/libnpcg_trace.so python tools/trace_ws.py

Per line warp: stages, cycles per stage (median), and where the solver's
stage time goes (ring read + full wait vs steps); per helper: how far the
prepared stage leads the solver.
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
    n = 32 * 1024 * 3
    buf = (ctypes.c_longlong * n)()
    rc = lib.npcg_debug_line_trace(buf, n)
    t = np.frombuffer(buf, dtype=np.int64).reshape(32, 1024, 3).astype(float)
    live = t[:, :, 0] > 0
    t0 = t[live][:, 0].min() if live.any() else 0
    print("rc", rc)
    for w in range(8):
        js = np.flatnonzero(live[w])
        if len(js) < 2:
            continue
        s = t[w, js] - t0
        per = np.median(np.diff(s[:, 0]))
        wait = np.median(s[:, 1] - s[:, 0])
        work = np.median(s[:, 2] - s[:, 1])
        print(f"line warp {w}: stages {len(js)} first {s[0,0]:.0f} last {s[-1,2]:.0f} | per stage {per:.0f} "
              f"(ring+full wait {wait:.0f}, steps {work:.0f}) | max wait {np.max(s[:,1]-s[:,0]):.0f}")
        h = w + 8
        hj = np.flatnonzero(live[h])
        if len(hj):
            hs = t[h, hj] - t0
            common = np.intersect1d(js, hj)
            lead = [t[w, j, 0] - t[h, j, 1] for j in common]  # solver stage start - prepared
            land = [t[h, j, 1] - t[h, j, 0] for j in common]
            print(f"   helper {w}: prepared-ahead median {np.median(lead):.0f} min {np.min(lead):.0f}; "
                  f"prepare {np.median(land):.0f}")
    for w in range(4):
        js = np.flatnonzero(live[w])
        for ph, sel in (("fwd", js[: len(js) // 2]), ("bwd", js[len(js) // 2:])):
            a = t[w, sel]
            r = t[16 + w, sel]
            h = t[8 + w, sel]
            h3 = t[24 + w, sel]
            print(f"warp {w} {ph}: interval {np.median(np.diff(a[:,0])):.0f} ring {np.median(r[:,0]-a[:,0]):.0f} "
                  f"check {np.median(r[:,1]-r[:,0]):.0f} full {np.median(a[:,1]-r[:,1]):.0f} steps {np.median(a[:,2]-a[:,1]):.0f} "
                  f"| helper prepare {np.median(h3[:,0]-h[:,0]):.0f} +rtma {np.median(h[:,1]-h3[:,0]):.0f} "
                  f"landed-before-start {np.median(a[:,0]-h[:,0]):.0f}")
    # global critical path: first / last stamp per warp, per phase
    np.save(os.path.join(ROOT, "gpurun_out", "trace_ws.npy"), t)


if __name__ == "__main__":
    main()
