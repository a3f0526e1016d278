"""Multi-rank host logic on CPU (gloo, world size 2 and 3): the NCCL unique-id
bootstrap, the ownership partition and the per-step exchange plan (a slice
broadcast from each owner rebuilds the full array on every rank), and the
max/sum reductions bench.py uses for its timing.  The GPU data path of the same
plan is covered by tests/test_gpu_parity.py::test_rank_emulation_bitwise."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1109_5190_b200 import dist as bdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1109_5190_b200 import bh

        uid = bdist.share_nccl_id(bh.nccl_unique_id, dist)
        # every rank starts with only its own slice of the positions filled
        full = np.arange(n * 4, dtype=np.float32).reshape(n, 4)
        mine = np.full_like(full, np.nan)
        lo, hi = bdist.own_range(n, rank, world)
        mine[lo:hi] = full[lo:hi]
        buf = torch.from_numpy(mine)
        for root, a, b in bdist.exchange_plan(n, world):
            sl = buf[a:b].clone()
            dist.broadcast(sl, src=root)
            buf[a:b] = sl
        ok = bool(np.array_equal(buf.numpy(), full))
        tmax = bdist.reduce_scalar(10.0 + rank, dist, "max")
        tsum = bdist.reduce_scalar(1.0 + rank, dist, "sum")
        out_q.put((rank, uid, ok, tmax, tsum, (lo, hi)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 1001), (3, 30000)])
def test_gloo_bootstrap_partition_exchange(world, n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    uids = {r[1] for r in res}
    assert len(uids) == 1 and len(next(iter(uids))) == 128
    assert all(r[2] for r in res), "exchange plan did not rebuild the full array"
    assert all(r[3] == 10.0 + world - 1 for r in res)
    assert all(r[4] == sum(1.0 + k for k in range(world)) for r in res)
    ranges = [r[5] for r in res]
    assert ranges[0][0] == 0 and ranges[-1][1] == n
    assert all(ranges[k][1] == ranges[k + 1][0] for k in range(world - 1))


def test_partition_edges():
    for n in (1, 2, 7, 4097):
        for world in range(1, min(n, 8) + 1):
            rs = [bdist.own_range(n, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(hi - lo in (n // world, n // world + 1) for lo, hi in rs)
            assert sum(hi - lo for _, lo, hi in bdist.exchange_plan(n, world)) == n


def test_cost_bounds_properties():
    """Equal-cost ownership split (bh_set_partition's input): covers [0, n),
    non-decreasing, every range within the library's velocity capacity, and
    per-rank costs within one particle's cost of total / P."""
    rng = np.random.default_rng(0)
    for n, world in [(1000, 2), (30001, 3), (50000, 8), (17, 4)]:
        costs = rng.integers(100, 3000, size=n).astype(np.float64)
        costs[: n // 5] *= 4  # a dense region
        b = bdist.cost_bounds(costs, world)
        assert b[0] == 0 and b[-1] == n and len(b) == world + 1
        assert all(b[i] <= b[i + 1] for i in range(world))
        cap = min(n, 2 * (-(-n // world)) + 1)
        assert all(b[i + 1] - b[i] <= cap for i in range(world))
        per = np.array([costs[b[i]:b[i + 1]].sum() for i in range(world)])
        assert per.max() - costs.sum() / world <= costs.max() + 1e-9 or n < 4 * world
        assert b == bdist.cost_bounds(costs.copy(), world)  # deterministic
    # equal costs give the even split
    assert bdist.cost_bounds(np.ones(12), 3) == [0, 4, 8, 12]


class _FakeBH:
    """Stands in for BarnesHut in the host-side rebalance: an own slice of
    costs and velocities over a known global array."""

    def __init__(self, n, rank, world, costs, vel):
        self.lo, self.hi = bdist.own_range(n, rank, world)
        self.costs, self.vel = costs, vel
        self.got = None

    def get_stats(self):
        return {"own_begin": self.lo, "own_end": self.hi}

    def get_own(self):
        return self.costs[self.lo:self.hi].astype(np.uint32), self.vel[self.lo:self.hi]

    def get_own_cost(self):  # the walk-trip costs (dist.rebalance's default)
        return self.costs[self.lo:self.hi].astype(np.uint32)

    def set_partition(self, bounds, vel_own):
        self.got = (list(bounds), np.array(vel_own))


def test_time_scaled_costs():
    """dist.time_scaled: a rank's costs rescaled to its measured walk time.
    Two ranks with equal summed costs but rank 1 twice as slow per unit:
    after rescaling, the equal-cost split moves work from rank 1 to rank 0
    so that the predicted times (cost x the rank's time per unit) equalise."""
    c = np.full(1000, 3.0)
    t = bdist.time_scaled(c, 6.0)
    assert np.isclose(t.sum(), 6.0) and np.allclose(t, t[0])
    assert np.array_equal(bdist.time_scaled(c, None), c)
    assert np.array_equal(bdist.time_scaled(np.zeros(5), 2.0), np.zeros(5))
    # per-unit speeds 1 (rank 0's half) and 2 (rank 1's half), equal costs
    n = 2000
    costs = np.ones(n)
    walk = [1000.0, 2000.0]  # measured ms of the halves
    scaled = np.concatenate([bdist.time_scaled(costs[:1000], walk[0]), bdist.time_scaled(costs[1000:], walk[1])])
    b = bdist.cost_bounds(scaled, 2)
    t0 = scaled[: b[1]].sum()
    t1 = scaled[b[1]:].sum()
    assert b[1] > 1000 and abs(t0 - t1) <= scaled.max() + 1e-9


def _rebalance_worker(rank, world, port, n, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(5)
        costs = rng.integers(1, 1000, size=n)
        vel = rng.standard_normal((n, 3)).astype(np.float32)
        bh = _FakeBH(n, rank, world, costs, vel)
        bounds = bdist.rebalance(bh, dist)
        b, v = bh.got
        ok = (b == list(bounds) == bdist.cost_bounds(costs, world)
              and np.array_equal(v, vel[b[rank]:b[rank + 1]]))
        out_q.put((rank, ok, b))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 1001), (3, 5000)])
def test_gloo_rebalance_host_logic(world, n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rebalance_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res)
    assert len({tuple(b) for _, _, b in res}) == 1  # every rank holds the same bounds
