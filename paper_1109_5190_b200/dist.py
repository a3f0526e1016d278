"""Host-side multi-GPU plumbing: ownership ranges, the NCCL
bootstrap through torch.distributed, and max/sum reductions over ranks.

The data path itself is in libbh.so: every rank holds the full position array,
builds the same tree, walks and integrates its own contiguous Morton range and
then broadcasts that slice to every other rank (api.cu `exchange`, a grouped
ncclBroadcast per owner) -- or, with share_replicas / bh_set_peers, stores
each new position straight into every rank's replica from the walk epilogue.
This module only mirrors the partition rule and moves small host objects; it
is tested with the gloo backend on CPU (tests/test_dist_gloo.py) because this
environment has a single GPU.
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


def cost_bounds(costs, world: int):
    """Equal-cost ownership split: bounds[world + 1] over
    storage order such that every rank's summed cost is as close as possible to
    total / world.  Rank r ends at the first storage id whose inclusive cost
    prefix reaches (r + 1) total / world.  Pure function of the costs, so every
    rank computes the same bounds.  Each range is capped at the velocity
    capacity 2 ceil(n / world) + 1 of the library."""
    import numpy as np

    c = np.asarray(costs, dtype=np.float64)
    n = c.shape[0]
    cap = min(n, 2 * (-(-n // world)) + 1)
    pre = np.cumsum(c)
    total = pre[-1] if n else 0.0
    b = [0]
    for r in range(1, world):
        target = total * r / world
        e = int(np.searchsorted(pre, target, side="left")) + 1 if total > 0 else n * r // world
        e = max(b[-1], min(e, n))
        e = min(e, b[-1] + cap)                      # this rank's capacity
        e = max(e, n - cap * (world - r))            # the remaining ranks' capacity
        b.append(e)
    b.append(n)
    return b


def time_scaled(costs, walk_ms):
    """One rank's per-particle costs rescaled so that they sum to the rank's
    measured walk time (ms per step): the equal-cost split of the rescaled
    costs then balances measured time, not a proxy -- time per walk trip
    differs between Morton ranges.  Unchanged without a time
    or with zero costs."""
    import numpy as np

    c = np.asarray(costs, dtype=np.float64)
    tot = float(c.sum())
    if walk_ms is None or not (walk_ms > 0.0) or not (tot > 0.0):
        return c
    return c * (float(walk_ms) / tot)


def rebalance(bh, dist, device=None, cost="trips", walk_ms=None):
    """Collective: gather every rank's per-particle costs and velocities,
    compute equal-cost bounds, and hand each rank its new range and velocities
    (bh_set_partition).  Returns the bounds.  cost = "trips": the last walk's
    loop trips of each particle's group (bh_get_own_cost: walk time), or
    "interactions": its interaction count (bh_get_own).  walk_ms (this rank's
    measured walk time per step, e.g. from bh_get_profile): the costs are
    rescaled to it first (time_scaled), so repeated calls converge on equal
    measured walk times."""
    import numpy as np
    import torch

    world = dist.get_world_size()
    st = bh.get_stats()
    lo, hi = int(st["own_begin"]), int(st["own_end"])
    cnt, vel = bh.get_own()
    if cost == "trips":
        cnt = bh.get_own_cost()
    cnt = time_scaled(cnt, walk_ms)
    sizes = [None] * world
    dist.all_gather_object(sizes, (lo, hi))
    m = max(h - l for l, h in sizes)
    pad_c = torch.zeros(m, dtype=torch.float64, device=device)
    pad_v = torch.zeros((m, 3), dtype=torch.float32, device=device)
    pad_c[: hi - lo] = torch.from_numpy(np.asarray(cnt, dtype=np.float64)).to(device)
    pad_v[: hi - lo] = torch.from_numpy(vel).to(device)
    all_c = [torch.empty_like(pad_c) for _ in range(world)]
    all_v = [torch.empty_like(pad_v) for _ in range(world)]
    dist.all_gather(all_c, pad_c)
    dist.all_gather(all_v, pad_v)
    costs = np.concatenate([all_c[r][: h - l].cpu().numpy() for r, (l, h) in enumerate(sizes)])
    vels = np.concatenate([all_v[r][: h - l].cpu().numpy() for r, (l, h) in enumerate(sizes)])
    bounds = cost_bounds(costs, world)
    me = dist.get_rank()
    bh.set_partition(bounds, vels[bounds[me]:bounds[me + 1]])
    return bounds


def share_replicas(bh, dist):
    """Collective: the fused exchange's plumbing (bh_set_peers).  Every rank
    exports its workspace as a CUDA IPC handle (torch.multiprocessing's
    reduce_tensor), all-gathers the handles with pos4's offset inside the
    workspace, opens the other ranks' workspaces (peer memory, mapped with
    lazy peer access) and hands the library every rank's pos4 address.  The
    opened mappings are kept on `bh` for as long as the peers are set."""
    from torch.multiprocessing.reductions import reduce_tensor

    world, me = dist.get_world_size(), dist.get_rank()
    off = bh.pos4_ptr() - bh.workspace.data_ptr()
    fn, args = reduce_tensor(bh.workspace)
    objs = [None] * world
    dist.all_gather_object(objs, (fn, args, off))
    ptrs, keep = [], []
    for r, (f, a, o) in enumerate(objs):
        if r == me:
            ptrs.append(bh.pos4_ptr())
            continue
        t = f(*a)
        keep.append(t)
        ptrs.append(t.data_ptr() + o)
    bh._peer_workspaces = keep
    bh.set_peers(ptrs)
    return ptrs


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
