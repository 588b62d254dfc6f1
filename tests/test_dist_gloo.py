"""Multi-process (world_size 2, gloo, CPU) checks of the N>1 host logic:
ranks get disjoint right-hand-side streams on one shared mesh, every rank
agrees on the job size, and the reported time is the max over ranks. The
data path itself has no collective (weak scaling of independent solves)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    import bench
    prob, model = bench.workload(k=12, batch=4, rank=rank)
    # shared mesh, distinct right-hand sides
    pat = torch.tensor([float(prob.A.values.sum()), float(prob.A.nnz)], dtype=torch.float64)
    pats = [torch.zeros_like(pat) for _ in range(world)]
    dist.all_gather(pats, pat)
    rhs = torch.from_numpy(prob.rhs.copy())
    rhss = [torch.zeros_like(rhs) for _ in range(world)]
    dist.all_gather(rhss, rhs)
    # max-over-ranks timing as bench.py does it
    t = torch.tensor([1.0 + rank], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    out[rank] = {
        "same_mesh": all(torch.equal(p, pats[0]) for p in pats),
        "distinct_rhs": not torch.equal(rhss[0], rhss[1]),
        "max_time": float(t.item()),
        "units": prob.rhs.shape[1] * world,
    }
    dist.destroy_process_group()


def test_two_rank_sharding_and_timing():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    for r in (0, 1):
        assert out[r]["same_mesh"]
        assert out[r]["distinct_rhs"]
        assert out[r]["max_time"] == 2.0
        assert out[r]["units"] == 8


def test_rank_streams_are_disjoint_and_reproducible():
    from paper_2305_16432_b200 import inputs
    a = inputs.poisson_2d(k=10, batch=3, first=0)
    b = inputs.poisson_2d(k=10, batch=3, first=3)
    c = inputs.poisson_2d(k=10, batch=6, first=0)
    np.testing.assert_array_equal(a.A.values, b.A.values)  # one mesh for every rank
    np.testing.assert_array_equal(c.rhs[:, :3], a.rhs)
    np.testing.assert_array_equal(c.rhs[:, 3:], b.rhs)  # rank 1's batch = streams 3..5
    assert not np.allclose(a.rhs, b.rhs)
