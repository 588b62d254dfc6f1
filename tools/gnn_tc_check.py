"""tcgen05 edge update vs the FFMA tiles vs the oracle: the GNN's raw edge
outputs M at latent 64 (config-2 mesh at size K), relative error of each
against the fp64 oracle, and the device GNN time of each path."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run_one():
    import torch
    import bench
    from paper_2305_16432_b200 import gnn
    k = int(os.environ.get("K", "64"))
    prob, model = bench.workload(k, 4)
    A = prob.A
    b = torch.from_numpy(prob.rhs[:, :1].copy()).cuda()
    pat, S, D, M, _ = gnn._gnn_device(model, A, b, want_edges=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        gnn._gnn_device(model, A, b)
    e1.record()
    e1.synchronize()
    np.save(os.environ["OUT"], M.cpu().numpy().reshape(-1))
    print("ms", e0.elapsed_time(e1) / 5)


def main():
    if os.environ.get("OUT"):
        return run_one()
    import bench
    from oracle import port
    k = int(os.environ.get("K", "64"))
    prob, model = bench.workload(k, 4)
    A = prob.A
    g = port.graph_from_system(port.Csr(A.n, A.row_ptr, A.col_idx, A.values), prob.rhs[:, 0])
    hp = port.Hyper(l=1, h=64, n_mp=5, l_mp=1, h_mp=64, width=64)
    ref, _ = port.gnn_run(hp, model.params, g)
    for tc in ("0", "1"):
        out = f"/tmp/gnn_M_{tc}.npy"
        r = subprocess.run([sys.executable, __file__], env={**os.environ, "OUT": out, "NPCG_GNN_TC": tc},
                           capture_output=True, text=True, timeout=300)
        print("tc", tc, r.stdout.strip(), r.stderr.strip()[-400:])
        M = np.load(out)
        print(f"   rel err vs oracle {np.linalg.norm(M - ref) / np.linalg.norm(ref):.3e}  max abs {np.abs(M - ref).max():.3e}")


if __name__ == "__main__":
    main()
