"""Compare the line-order path against the level path (NPCG_NO_LINES) on the
config-1 workload: iterations per system and solution difference."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run():
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    import bench
    from paper_2305_16432_b200 import gnn, pcg
    k = int(os.environ.get("K", "256"))
    B = int(os.environ.get("B", "64"))
    prob, model = bench.workload(k, B)
    rhs = torch.from_numpy(prob.rhs).cuda()
    opts = pcg.SolveOptions(thresholds=(bench.CFG["rtol"],), max_iter=int(os.environ.get("MAXIT", "1500")))
    P = gnn.build_learned(model, prob.A, rhs[:, 0])
    X, reps = pcg.pcg_solve_batch(prob.A, rhs, P, opts)
    np.save(os.environ["OUT"], np.concatenate([np.array([[r.iterations for r in reps]], dtype=float),
                                               X.cpu().numpy()]))


if __name__ == "__main__":
    if len(sys.argv) > 1:
        run()
    else:
        import numpy as np
        env = dict(os.environ)
        subprocess.run([sys.executable, __file__, "x"], env=dict(env, OUT="/tmp/a.npy"), check=True)
        subprocess.run([sys.executable, __file__, "x"], env=dict(env, OUT="/tmp/b.npy", NPCG_NO_LINES="1"), check=True)
        a, b = np.load("/tmp/a.npy"), np.load("/tmp/b.npy")
        print("iters lines :", a[0].astype(int).tolist())
        print("iters levels:", b[0].astype(int).tolist())
        d = np.abs(a[1:] - b[1:]).max(axis=0) / np.abs(b[1:]).max(axis=0)
        print("rel x diff per system:", np.array2string(d, precision=2))
