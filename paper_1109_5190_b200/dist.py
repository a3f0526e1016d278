"""Host-side multi-GPU plumbing: ownership ranges, the NCCL
bootstrap through torch.distributed, and max/sum reductions over ranks.

The data path itself is in libbh.so: every rank holds the full position array,
builds the same tree, walks and integrates its own contiguous Morton range and
then broadcasts that slice to every other rank (api.cu `exchange`, a grouped
ncclBroadcast per owner).  This module only mirrors the partition rule and
moves small host objects; it is tested with the gloo backend on CPU
(tests/test_dist_gloo.py) because this environment has a single GPU.
"""
from __future__ import annotations

import os


def env_rank():
    """(rank, world, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def own_range(n: int, rank: int, world: int):
    """Storage ids [lo, hi) owned by `rank` (api.cu: own_lo = n r / P)."""
    return n * rank // world, n * (rank + 1) // world


def exchange_plan(n: int, world: int):
    """The grouped broadcast of one step: (root, lo, hi) per non-empty slice."""
    out = []
    for r in range(world):
        lo, hi = own_range(n, r, world)
        if hi > lo:
            out.append((r, lo, hi))
    return out


def share_nccl_id(make_id, dist) -> bytes:
    """Rank 0 makes the 128-byte ncclUniqueId; every rank receives it."""
    obj = [make_id() if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def reduce_scalar(x: float, dist, op: str, device=None) -> float:
    """max / sum of a host scalar over all ranks (device tensor for NCCL)."""
    import torch

    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())
