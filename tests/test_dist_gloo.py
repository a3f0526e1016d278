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
