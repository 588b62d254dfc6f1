"""Timeline of the warp-specialised line solve (block 0), from a library
built with -DNPCG_LINE_TRACE:

    make -C paper_2305_16432_b200/csrc EXTRA=-DNPCG_LINE_TRACE
    python tools/trace_line.py            # runs one profiled config-1 solve

Prints per-batch cycle gaps between consumer and producer events.
"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

EV = ["c_full_wait", "c_full_done", "c_batch_end", "p_start", "p_drained", "p_rhs_done", "p_mbar_done", "-",
      "c_q0", "c_q1", "c_q2", "c_q3", "p_waitread", "p_issued", "cfg", "-"]


def main():
    import torch
    from paper_2305_16432_b200 import _native, gnn, inputs, pcg
    k = int(os.environ.get("PROBE_K", "256"))
    B = int(os.environ.get("PROBE_B", "64"))
    which = os.environ.get("TRACE_DIR", "fwd")
    prob = inputs.poisson_2d(k=k, batch=B)
    A = prob.A
    rng = np.random.default_rng(0)
    P = gnn.assemble_preconditioner(rng.uniform(-0.2, 0.2, A.strict_lower().nnz), A)
    rhs = torch.from_numpy(prob.rhs).cuda()
    # one iteration: the forward solve of the last launch is what the buffer holds
    opts = pcg.SolveOptions(thresholds=(1e-8,), max_iter=int(os.environ.get("TRACE_ITERS", "3")))
    pcg.pcg_solve_batch(A, rhs, P, opts, with_history=False)
    torch.cuda.synchronize()
    lib = _native.load_library()
    buf = (ctypes.c_longlong * (16 * 2048))()
    rc = lib.npcg_debug_line_trace(buf, 16 * 2048)
    t = np.frombuffer(buf, dtype=np.int64).reshape(16, 2048)
    nb = int((t[1] > 0).sum())
    ev = [e for e in range(16) if e not in (7, 14, 15)]
    t0 = t[ev, :nb][t[ev, :nb] > 0].min()
    rel = np.where(t[:, :nb] > 0, t[:, :nb] - t0, -1)
    print("rc", rc, "batches", nb, "(last launch =", which, ")")
    print("NS A nb max_slots T W MD smem:", list(t[14, :8]))
    print("batch " + " ".join(f"{e:>12s}" for e in EV))
    for j in list(range(0, min(nb, 12))) + list(range(nb // 2, nb // 2 + 8)):
        print(f"{j:5d} " + " ".join(f"{rel[e, j]:12d}" for e in range(7)))
    if nb > 20:
        mid = slice(nb // 4, 3 * nb // 4)
        per = np.diff(rel[1, mid]).mean()
        print("cycles per batch (consumer, mid):", round(per, 1))
        ns = np.diff(t[15, :nb]).astype(float)
        print("ns per batch (globaltimer, mid):", round(ns[nb // 4:3 * nb // 4].mean(), 1), " whole solve us:",
              round((t[15, nb - 1] - t[15, 0]) / 1e3, 1), " clock GHz:", round(per / ns[nb // 4:3 * nb // 4].mean(), 3))
        for e in list(range(7)) + list(range(8, 14)):
            print(f"  {EV[e]:>14s} - c_full_done: {np.mean(rel[e, mid] - rel[1, mid]):10.1f}")


if __name__ == "__main__":
    main()
