"""Multi-GPU batch parallelism: independent systems /
right-hand sides are split into contiguous shards, one per rank (one
process per GPU); every rank solves its shard with no communication inside
the PCG loop, and the results -- x, iteration counts, status -- are
gathered to one rank at the end over NCCL (NVLink / NVSwitch), in global
system order.

The reference has no distribution at all; its only concurrency is a thread
pool over independent benchmark cells (pkg/src/pcgkit/bench.py:149-153),
and SPEC.md:296 allows independent solves over shared immutable A and P --
the contract this module relies on. Works with any torch.distributed
backend (nccl on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def shard(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous range [lo, hi) of `total` units owned by `rank`; shard
    sizes differ by at most one, lower ranks take the remainder."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank must lie in [0, world)")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


@dataclass
class Gathered:
    """Rank-0 view of a sharded batch solve, in global system order."""
    X: object                # (n, total) tensor on the gathering rank's device
    iterations: np.ndarray   # (total,)
    status: np.ndarray       # (total,) NPCG status codes
    converged: np.ndarray    # (total,) bool


def _dist():
    import torch.distributed as dist
    return dist


def gather_solutions(X_local, iterations, status, total: int, dst: int = 0, group=None):
    """Gather every rank's (n, B_r) solution block plus its per-system
    iteration counts and status to rank `dst` (global order = rank order,
    matching shard()). Returns a Gathered on `dst`, None elsewhere.

    The blocks travel as equal-sized padded shards (shards differ by at most
    one system) in one gather to `dst` -- only the gathering rank receives
    the solutions; a small side tensor carries each column's iteration
    count, status and liveness.
    """
    import torch
    dist = _dist()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = X_local.device
    n, b_local = X_local.shape
    width = -(-total // world)  # ceil: the widest shard
    lo, hi = shard(total, world, rank)
    if hi - lo != b_local:
        raise ValueError(f"rank {rank} holds {b_local} systems, its shard is {hi - lo}")
    # columns -> rows so a shard is one contiguous block; padded to `width`
    blk = torch.zeros((width, n), dtype=X_local.dtype, device=dev)
    blk[:b_local] = X_local.t()
    meta = torch.zeros((width, 3), dtype=torch.int64, device=dev)
    meta[:b_local, 0] = torch.as_tensor(np.asarray(iterations, dtype=np.int64), device=dev)
    meta[:b_local, 1] = torch.as_tensor(np.asarray(status, dtype=np.int64), device=dev)
    meta[:b_local, 2] = 1  # live column
    if rank == dst:
        blks = [torch.empty_like(blk) for _ in range(world)]
        metas = [torch.empty_like(meta) for _ in range(world)]
    else:
        blks = metas = None
    dist.gather(blk, blks, dst=dst, group=group)
    dist.gather(meta, metas, dst=dst, group=group)
    if rank != dst:
        return None
    all_blk = torch.cat(blks)
    all_meta = torch.cat(metas)
    live = all_meta[:, 2].bool()
    X = all_blk[live].t().contiguous()
    m = all_meta[live].cpu().numpy()
    if X.shape[1] != total:
        raise RuntimeError("gathered shard widths do not add up to the batch")
    from . import _native
    return Gathered(X, m[:, 0].copy(), m[:, 1].copy(), m[:, 1] == _native.STATUS_CONVERGED)
