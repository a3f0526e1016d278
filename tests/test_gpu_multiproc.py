"""The multi-GPU step loop as TWO PROCESSES on one GPU (this environment has a
single B200): rank r of 2 owns a Morton range, builds the full tree, walks and
integrates its range; the K8 exchange is done over a gloo process group
through bh_get_pos4 / bh_set_pos4 (no NCCL communicator: nccl_comm = NULL), and
dist.rebalance runs on the real BarnesHut objects mid-run (equal-cost split
from the last walk's interaction counts).  The processes never wait on each
other inside a kernel (only host collectives), so sharing the GPU is safe.
The fused variant shares the replicas by CUDA IPC instead (dist.share_replicas:
the walk epilogue of each process stores into the other's pos4; NEXT-1).
Bar: every particle's position and velocity after 4 steps bitwise equal to the
P = 1 run, and within 1e-4 of the fp64 oracle (every
iteration needs all particles' positions)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

STEPS, REBALANCE_AT, N = 4, 2, 20000


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, out_q, fused=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    import bhgen
    from paper_1109_5190_b200 import BarnesHut
    from paper_1109_5190_b200 import dist as bdist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, p, v = bhgen.generate("cfg2", n=N)
        prm = bhgen.params("cfg2")
        bh = BarnesHut(m, p, v, device=0, rank=rank, world=world, nccl_comm=None, **prm)
        bounds = [N * r // world for r in range(world + 1)]
        moved = None
        if fused:  # K8 fused into K7: IPC-shared replicas (bh_set_peers)
            ptrs = bdist.share_replicas(bh, dist)
            assert len(set(ptrs)) == world
        for k in range(STEPS):
            if k == REBALANCE_AT:
                new = bdist.rebalance(bh, dist)  # all-gathers costs + velocities, bh_set_partition
                moved = new != bounds
                bounds = new
            if fused:
                # every rank builds from the old positions, then every rank's walk
                # stores its new positions into all replicas; host barriers order
                # the phases (a communicator would put them in the step's graph)
                bh.step_phase(0)
                bh.sync()
                dist.barrier()
                bh.step_phase(1)
                bh.sync()
                dist.barrier()
                continue
            bh.step(1)
            # K8 over gloo: every owner's slice of pos4 (x, y, z, m) to every rank
            mine = torch.from_numpy(bh.get_pos4(bounds[rank], bounds[rank + 1]))
            for r in range(world):
                sl = mine.clone() if r == rank else torch.empty((bounds[r + 1] - bounds[r], 4), dtype=torch.float32)
                dist.broadcast(sl, src=r)
                if r != rank:
                    bh.set_pos4(sl.numpy(), bounds[r], bounds[r + 1])
        pos, vel = bh.get_state()
        st = bh.get_stats()
        out_q.put((rank, pos, vel, (int(st["own_begin"]), int(st["own_end"])), bounds, moved))
        if fused:
            bh.set_peers(None)
            dist.barrier()  # nobody unmaps a replica another rank may still write
        bh.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fused", [False, True], ids=["gloo_exchange", "fused_peer_stores"])
def test_two_processes_one_gpu_gloo_exchange_and_rebalance(fused):
    import torch
    import torch.multiprocessing as mp

    import bhgen
    import oracle
    from paper_1109_5190_b200 import BarnesHut

    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, q, fused)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda t: t[0])
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    m, p, v = bhgen.generate("cfg2", n=N)
    prm = bhgen.params("cfg2")
    one = BarnesHut(m, p, v, **prm)
    one.build_tree()
    _, perm = one.get_keys()  # storage id -> user index (storage order = step-0 Morton order)
    one.step(STEPS)
    ref_pos, ref_vel = one.get_state()
    one.close()
    bounds = res[0][4]
    assert all(r[4] == bounds for r in res) and res[0][5], "the rebalance did not move the split"
    got_pos = np.full_like(ref_pos, np.nan)
    got_vel = np.full_like(ref_vel, np.nan)
    for rank, pos, vel, (lo, hi), _, _ in res:
        assert (lo, hi) == (bounds[rank], bounds[rank + 1])
        assert np.array_equal(pos, ref_pos)  # the replicated positions everywhere
        own = perm[lo:hi].astype(np.int64)
        got_pos[own] = pos[own]
        got_vel[own] = vel[own]
    assert np.array_equal(got_pos, ref_pos) and np.array_equal(got_vel, ref_vel)
    o = oracle.Oracle(m, p.astype(np.float64), v.astype(np.float64), **prm)
    o.step(STEPS)
    opos, ovel = o.state()
    err = np.linalg.norm(got_pos - opos, axis=1) / np.linalg.norm(opos, axis=1)
    assert err.max() < 1e-4
