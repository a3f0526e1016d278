"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle.

Bar (BASELINE.json north_star): Morton keys, sort permutation and tree topology
bit-exact; fp64 moments bit-exact (reading L14); interaction counts
integer-exact (the MAC decisions are exact); per-particle accelerations and
positions after the stated steps within 1e-4 relative error,
max_i |a_gpu - a_ref| / |a_ref| (reading L23).
"""
import os

import numpy as np
import pytest

import bhgen
import oracle

pytestmark = pytest.mark.gpu

TOL = 1e-4


@pytest.fixture(scope="module")
def BH():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_1109_5190_b200 import BarnesHut

    return BarnesHut


def relerr(a, ref):
    a = np.asarray(a, np.float64)
    ref = np.asarray(ref, np.float64)
    num = np.linalg.norm(a - ref, axis=1)
    den = np.linalg.norm(ref, axis=1)
    return np.where(den > 0, num / np.where(den > 0, den, 1), num)


def _oracle(m, p, v, prm):
    return oracle.Oracle(m, np.asarray(p, np.float64), None if v is None else np.asarray(v, np.float64), **prm).build()


def check_step0(bh, o, n, full_forces=True, targets=None):
    k, perm = bh.get_keys()
    ok, operm = o.keys()
    assert np.array_equal(k, ok), "Morton keys differ"
    assert np.array_equal(perm.astype(np.int64), operm), "sort permutation differs"
    lv, fi, co = bh.get_tree()
    olv, ofi, oco, oM, oMX = o.tree(with_moments=True)
    assert len(lv) == len(olv), f"node count {len(lv)} vs {len(olv)}"
    assert np.array_equal(lv, olv) and np.array_equal(fi, ofi) and np.array_equal(co, oco), "topology differs"
    M, MX = bh.get_moments()
    assert np.array_equal(M, oM) and np.array_equal(MX, oMX), "fp64 moments not bit-identical"
    acc = bh.compute_forces()
    cnt, total = bh.get_interactions()
    if targets is None:
        oacc, ocnt = o.forces()
        assert np.array_equal(cnt.astype(np.int64), ocnt), "interaction counts differ"
        assert total == int(ocnt.sum())
        err = relerr(acc, oacc)
    else:
        oacc, ocnt = o.forces(targets)
        assert np.array_equal(cnt[targets].astype(np.int64), ocnt), "interaction counts differ"
        err = relerr(acc[targets], oacc)
    assert err.max() < TOL, f"acceleration max rel err {err.max():.3e}"
    return acc, err


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2"])
def test_full_config_parity_free_running(BH, cfg):
    """cfg1 (1 step) and cfg2 (10 steps): step 0 bit-exact + forces, then the
    free-running trajectory (positions <= 1e-4 after the stated steps) and a
    teacher-forced check on the GPU's final state (reading L24)."""
    c = bhgen.CONFIGS[cfg]
    m, p, v = bhgen.generate(cfg)
    prm = bhgen.params(cfg)
    bh = BH(m, p, v, **prm)
    bh.build_tree()
    o = _oracle(m, p, v, prm)
    check_step0(bh, o, c.n)
    bh.step(c.steps)
    gpos, gvel = bh.get_state()
    o.step(c.steps)
    opos, ovel = o.state()
    perr = relerr(gpos, opos)
    assert perr.max() < TOL, f"positions after {c.steps} steps: {perr.max():.3e}"
    # teacher-forced: the oracle on the GPU's fp32 state reproduces keys/topology/forces
    bh.build_tree()
    ot = oracle.Oracle(m, gpos.astype(np.float64), gvel.astype(np.float64), **prm).build()
    check_step0(bh, ot, c.n)
    st = bh.get_stats()
    assert st["steps"] == c.steps


def test_cfg3_full_step0_and_stated_steps(BH):
    """cfg3 (2^20, theta = 0.7): step 0 bit-exact + forces over all N, then the
    BASELINE's 5 steps free-running on both sides: positions <= 1e-4."""
    m, p, v = bhgen.generate("cfg3")
    prm = bhgen.params("cfg3")
    bh = BH(m, p, v, **prm)
    bh.build_tree()
    o = _oracle(m, p, v, prm)
    check_step0(bh, o, m.shape[0])
    steps = bhgen.CONFIGS["cfg3"].steps
    bh.step(steps)
    o.step(steps)
    gpos, _ = bh.get_state()
    opos, _ = o.state()
    assert relerr(gpos, opos).max() < TOL


def check_tree_of_last_build(bh, o):
    """Keys, permutation and topology of the GPU's last build (the one bh_step
    made of the current state) bit-exact against an oracle built on that state."""
    k, perm = bh.get_keys()
    ok, operm = o.keys()
    assert np.array_equal(k, ok), "Morton keys differ"
    assert np.array_equal(perm.astype(np.int64), operm), "sort permutation differs"
    lv, fi, co = bh.get_tree()
    olv, ofi, oco = o.tree()
    assert np.array_equal(lv, olv) and np.array_equal(fi, ofi) and np.array_equal(co, oco), "topology differs"


@pytest.mark.parametrize("cfg", ["cfg4", "cfg5"])
def test_full_size_all_targets_and_stated_steps(BH, cfg):
    """BASELINE full sizes (N = 2^24, 2^26) in the bench's launch configuration.
    Step 0: keys / permutation / topology / fp64 moments bit-exact, interaction
    counts integer-exact and accelerations within 1e-4 over ALL N targets (the
    max over particles of the north-star gate).  Then the stated steps (5 /
    10) on the GPU, teacher-forced (reading L24): at every cfg4 step and at
    cfg5 steps 1, 5 and 10 the oracle is built on the GPU's state at step k
    and makes one leapfrog step of 4096 sampled particles -- positions and
    velocities at step k + 1 within 1e-4, their interaction counts exact, and
    the GPU's keys / permutation / topology of state k (the near-sorted sort
    at full size) bit-exact.  PAPER.md:461-463 (Fig. 2c: "compute the next
    iteration values"), 58-63."""
    c = bhgen.CONFIGS[cfg]
    m, p, v = bhgen.generate(cfg)
    prm = bhgen.params(cfg)
    n = m.shape[0]
    bh = BH(m, p, v, **prm)
    bh.build_tree()
    o = oracle.Oracle(m, p.astype(np.float64), v.astype(np.float64), k0=0, **prm).build()
    _, err = check_step0(bh, o, n)
    print(f"{cfg} step 0, all {n} targets: acc max rel {err.max():.3e}, p99 {np.quantile(err, 0.99):.3e}")
    rng = np.random.default_rng(7)
    targets = np.sort(rng.choice(n, 4096, replace=False))
    check_at = set(range(c.steps)) if cfg == "cfg4" else {0, 4, 9}
    pos, vel = p, v
    for k in range(c.steps):
        ok_ = None
        if k in check_at:
            ok_ = o if k == 0 else oracle.Oracle(m, pos.astype(np.float64), vel.astype(np.float64), k0=k, **prm)
            po, vo, ocnt = ok_.step_targets(targets)
        bh.step(1)
        pos1, vel1 = bh.get_state()
        if ok_ is not None:
            if k > 0:
                assert bh.get_stats()["near_sorted"] == 1
            check_tree_of_last_build(bh, ok_)
            cnt, _ = bh.get_interactions()
            assert np.array_equal(cnt[targets].astype(np.int64), ocnt), f"step {k}: interaction counts differ"
            pe, ve = relerr(pos1[targets], po), relerr(vel1[targets], vo)
            print(f"{cfg} step {k} -> {k + 1} (teacher-forced, 4096 targets): pos max rel {pe.max():.3e}, "
                  f"vel max rel {ve.max():.3e}")
            assert pe.max() < TOL and ve.max() < TOL, (k, pe.max(), ve.max())
            ok_.close()
        pos, vel = pos1, vel1


@pytest.mark.parametrize("n", [1, 2, 3, 31, 33, 4097, 5000])
def test_ragged_and_tiny_sizes(BH, n):
    m, p, v = bhgen.generate("cfg2", n=n)
    prm = bhgen.params("cfg2")
    bh = BH(m, p, v, **prm)
    bh.build_tree()
    o = _oracle(m, p, v, prm)
    if n == 1:
        a = bh.compute_forces()
        assert np.all(a == 0)
        k, perm = bh.get_keys()
        assert list(perm) == [0]
        return
    check_step0(bh, o, n)
    bh.step(3)
    o.step(3)
    assert relerr(bh.get_state()[0], o.state()[0]).max() < TOL


@pytest.mark.parametrize("theta", [0.5, 0.7])
def test_eps_below_fp32_square(BH, theta):
    """eps > 0 whose fp32 square is zero (eps = 1e-25): the walk's fast paths
    that rely on a finite unmasked force (no per-visit containment test, the
    force mask on r2) must not run, since rsqrt(0) is inf and 0 x inf a NaN
    (api.cu eps2_normal); forces and 2 steps still match the oracle."""
    n = 6000
    m, p, v = bhgen.generate("cfg3", n=n)
    prm = dict(theta=theta, eps=1e-25, G=1.0, dt=1e-6)
    bh = BH(m, p, v, walk_group=69, **prm)
    bh.build_tree()
    o = _oracle(m, p, v, prm)
    check_step0(bh, o, n)
    bh.step(2)
    o.step(2)
    pos = bh.get_state()[0]
    assert np.isfinite(pos).all()
    assert relerr(pos, o.state()[0]).max() < TOL


def test_buckets_duplicates_coincident(BH):
    rng = np.random.default_rng(1)
    base = rng.random((3000, 3)).astype(np.float32)
    pos = np.vstack([base, base[rng.integers(0, 3000, 200)], np.tile(base[:1], (40, 1))])
    pos = pos[rng.permutation(pos.shape[0])]
    n = pos.shape[0]
    m = (rng.random(n) + 0.5).astype(np.float32)
    prm = dict(theta=0.6, eps=1e-2, G=1.0, dt=1e-3)
    bh = BH(m, pos, None, **prm)
    bh.build_tree()
    o = _oracle(m, pos, None, prm)
    check_step0(bh, o, n)
    lv, fi, co = bh.get_tree()
    assert np.any((lv == 21) & (co >= 2)), "expected level-21 buckets"
    # all particles coincident: L = 0, 22-node chain ending in a bucket
    pos = np.tile(np.float32([[0.5, -1.0, 2.0]]), (1000, 1))
    bh = BH(np.ones(1000, np.float32), pos, None, **prm)
    bh.build_tree()
    lv, fi, co = bh.get_tree()
    assert list(lv) == list(range(22)) and np.all(co == 1000)
    a = bh.compute_forces()
    assert np.all(a == 0)
    cnt, _ = bh.get_interactions()
    assert np.all(cnt == 999)


@pytest.mark.parametrize("k", [40, 3000, 9000])
def test_long_equal_key_runs(BH, k):
    """Equal-key runs longer than 32 go to k_long_runs (bitonic tiles of 4096,
    then pairwise merges by rank): k particles coincident with one of 2000
    others, the coincident ones scattered through the user order and moved
    onto the cluster point only after a step (so the run arrives in storage
    order, not user order).  Keys / permutation / topology bit-exact against
    the oracle (ties by user index, reading L13) at create and at the next
    build, counts exact, forces within 1e-4."""
    rng = np.random.default_rng(k)
    n = 2000 + k
    pos = rng.random((n, 3)).astype(np.float32)
    m = (rng.random(n) + 0.5).astype(np.float32)
    idx = rng.permutation(n)[:k]
    pos[idx] = pos[idx[0]]  # one cluster of k coincident particles, scattered in user order
    prm = dict(theta=0.6, eps=1e-2, G=1.0, dt=1e-3)
    bh = BH(m, pos, None, **prm)
    bh.build_tree()
    o = _oracle(m, pos, None, prm)
    check_step0(bh, o, n)
    # the cluster re-forms from particles whose storage order is not their
    # user order: swap the cluster with particles elsewhere and rebuild
    pos2 = pos.copy()
    other = np.setdiff1d(np.arange(n), idx)[: k // 2]
    pos2[other] = pos[idx[0]]
    pos2[idx[: k // 2]] = rng.random((k // 2, 3)).astype(np.float32)
    bh.set_state(m, pos2, None)
    bh.build_tree()
    o2 = _oracle(m, pos2, None, prm)
    check_step0(bh, o2, n)


def test_faces_and_theta0_direct(BH):
    rng = np.random.default_rng(2)
    pos = (rng.integers(0, 5, size=(2000, 3)) * 0.25).astype(np.float32) + rng.random((2000, 3)).astype(np.float32) * 1e-3
    pos[:10] = np.float32([[0, 0, 0]]) + 0  # on the lower faces
    m = np.full(2000, 1 / 2000, np.float32)
    prm = dict(theta=0.0, eps=1e-3, G=1.0, dt=1e-3)
    bh = BH(m, pos, None, **prm)
    bh.build_tree()
    o = _oracle(m, pos, None, prm)
    acc, _ = check_step0(bh, o, 2000)
    cnt, _ = bh.get_interactions()
    ref = oracle.direct(m, pos, 1e-3)
    assert relerr(acc, ref).max() < TOL and np.all(cnt == 1999)


def test_errors(BH):
    from paper_1109_5190_b200 import BhError

    m = np.ones(4, np.float32)
    pos = np.float32([[0, 0, 0], [1, 0, 0], [1, 0, 0], [0, 1, 0]])
    bh = BH(m, pos, None, theta=0.5, eps=0.0)
    with pytest.raises(BhError) as e:
        bh.compute_forces()  # before bh_build_tree
    assert e.value.code == -4
    bh.build_tree()
    with pytest.raises(BhError) as e:
        bh.compute_forces()  # eps == 0 and coincident pair
    assert e.value.code == -5
    bad = pos.copy()
    bad[2, 1] = np.nan
    with pytest.raises(BhError) as e:
        BH(m, bad, None, theta=0.5, eps=0.1)
    assert e.value.code == -5
    with pytest.raises(BhError) as e:
        BH(m, pos, None, theta=-1.0, eps=0.1)
    assert e.value.code == -1
    # node capacity too small for the tree -> BH_ERR_OOM
    mm, pp, _ = bhgen.generate("cfg1")
    bh = BH(mm, pp, None, theta=0.5, eps=1e-3, node_capacity=4097)
    bh.build_tree()
    with pytest.raises(BhError) as e:
        bh.sync()
    assert e.value.code == -3


@pytest.mark.parametrize("cfg,group", [(c, g) for c in ("cfg2", "cfg3") for g in (66, 67, 68, 69, 70)])
def test_walk_group_sizes(BH, cfg, group):
    """The traversal-sharing group shape (8 / 4 / 2 lanes x 2 targets, 2 / 1
    lanes x 4 targets) never changes a MAC
    decision: interaction counts integer-equal to the oracle's; a target's fp32
    block sums follow its group's walk, so forces agree to rounding (and with
    the oracle within 1e-4).  cfg2: theta = 0.5 (containment test elided);
    cfg3: theta = 0.7 (containment folded into the thresholds)."""
    m, p, v = bhgen.generate(cfg, n=20000)
    prm = bhgen.params(cfg)
    a = BH(m, p, v, **prm)
    a.build_tree()
    ref = a.compute_forces()
    b = BH(m, p, v, walk_group=group, **prm)
    b.build_tree()
    got = b.compute_forces()
    assert np.array_equal(a.get_interactions()[0], b.get_interactions()[0])
    assert relerr(got, ref).max() < 1e-5
    o = _oracle(m, p, v, prm)
    oacc, ocnt = o.forces()
    assert np.array_equal(b.get_interactions()[0].astype(np.int64), ocnt)
    assert relerr(got, oacc).max() < TOL


@pytest.mark.parametrize("cfg,group,variant", [("cfg3", 68, ""), ("cfg3", 67, ""), ("cfg3", 66, ""), ("cfg3", 69, ""),
                                               ("cfg3", 70, ""),
                                               ("cfg5", 68, ""), ("cfg3", 68, "massless"),
                                               ("cfg3", 68, "scaled")])
def test_containment_fold_vs_test(BH, cfg, group, variant, monkeypatch):
    """theta >= 0.57: containment folded into T_acc through the nodes' bounding
    radii (no per-visit test) == the walk that tests containment per visit:
    identical interaction counts; forces bitwise equal when no extra target
    fell back to the exact re-walk (else within fp32 rounding).  Variants:
    massless particles and a massless cluster; physical-scale units (masses
    x 1e25, G x 1e-25: M_j |com - com_j| overflows fp32 in the radius, ADVICE
    r1), both also against the oracle."""
    m, p, v = bhgen.generate(cfg, n=30000)
    prm = bhgen.params(cfg)
    massless = variant == "massless"
    if variant == "scaled":
        m = (m.astype(np.float64) * 1e25).astype(np.float32)
        prm = dict(prm, G=prm.get("G", 1.0) * 1e-25)
    if massless:  # massless particles and a massless cluster (no com to bound a node by)
        m = m.copy()
        m[::97] = 0.0
        p = p.copy()
        p[:50] = p[0] + np.float32(1e-4) * np.arange(50, dtype=np.float32)[:, None]
        m[:50] = 0.0
    a = BH(m, p, v, walk_group=group, **prm)  # fold (default for theta >= 0.57, eps > 0)
    a.build_tree()
    fa = a.compute_forces()
    ra = a.get_stats()["redo_targets"]
    monkeypatch.setenv("BH_NO_CONT_FOLD", "1")
    b = BH(m, p, v, walk_group=group, **prm)
    b.build_tree()
    fb = b.compute_forces()
    rb = b.get_stats()["redo_targets"]
    assert np.array_equal(a.get_interactions()[0], b.get_interactions()[0])
    if ra == rb:
        assert np.array_equal(fa, fb)
    else:  # the extra fallbacks sum their tails in fp64: per-particle relative difference
        rel = np.linalg.norm(fa.astype(np.float64) - fb, axis=1) / np.linalg.norm(fb.astype(np.float64), axis=1)
        assert rel.max() <= 1e-5
    if variant:  # and the folded walk against the oracle (counts exact, forces 1e-4)
        o = _oracle(m, p, v, prm)
        oacc, ocnt = o.forces()
        assert np.array_equal(a.get_interactions()[0].astype(np.int64), ocnt)
        assert relerr(fa, oacc).max() < TOL


@pytest.mark.parametrize("world,group", [(2, 0), (3, 0), (3, 69), (2, 70)])
def test_rank_emulation_bitwise(BH, world, group):
    """Multi-GPU path emulated on one GPU (no NCCL): each rank walks the P = 1
    groups that hold its particles, so its forces and one-step positions are
    bitwise the P = 1 ones (every group shape: the fp32 block sums follow the
    group's walk)."""
    m, p, v = bhgen.generate("cfg2", n=30000)
    prm = dict(bhgen.params("cfg2"), walk_group=group)
    one = BH(m, p, v, **prm)
    one.build_tree()
    ref = one.compute_forces()
    one.step(1)
    ref_pos, ref_vel = one.get_state()
    got = np.full_like(ref, np.nan)
    got_pos = np.full_like(ref, np.nan)
    got_vel = np.full_like(ref, np.nan)
    for r in range(world):
        bh = BH(m, p, v, rank=r, world=world, **prm)
        st = bh.get_stats()
        lo, hi = st["own_begin"], st["own_end"]
        assert hi > lo
        bh.build_tree()
        # storage order == step-0 Morton order, so the owned users are perm[lo:hi]
        _, perm = bh.get_keys()
        own = perm[lo:hi].astype(np.int64)
        a = bh.compute_forces()
        got[own] = a[own]
        bh.step(1)
        pos, vel = bh.get_state()
        got_pos[own] = pos[own]
        got_vel[own] = vel[own]
    assert not np.isnan(got).any()
    assert np.array_equal(got, ref)
    assert np.array_equal(got_pos, ref_pos) and np.array_equal(got_vel, ref_vel)


def test_device_pointer_paths(BH):
    import torch

    m, p, v = bhgen.generate("cfg1")
    prm = bhgen.params("cfg1")
    dm, dp, dv = (torch.from_numpy(x).cuda() for x in (m, p, v))
    bh = BH(dm, dp, dv, **prm)
    bh.build_tree()
    out = torch.empty((m.shape[0], 3), dtype=torch.float32, device="cuda")
    bh.compute_forces(out)
    host = BH(m, p, v, **prm)
    host.build_tree()
    assert np.array_equal(out.cpu().numpy(), host.compute_forces())
    bh.step(1)
    po = torch.empty_like(out)
    vo = torch.empty_like(out)
    bh.get_state(po, vo)
    host.step(1)
    hp, hv = host.get_state()
    assert np.array_equal(po.cpu().numpy(), hp) and np.array_equal(vo.cpu().numpy(), hv)
    bh.set_state(dm, dp, dv)
    bh.step(1)
    bh.get_state(po, vo)
    assert np.array_equal(po.cpu().numpy(), hp)
    # mass None keeps the masses (device and host inputs)
    bh.set_state(None, dp, dv)
    bh.step(1)
    bh.get_state(po, vo)
    assert np.array_equal(po.cpu().numpy(), hp)
    host.set_state(None, p, v)
    host.step(1)
    assert np.array_equal(host.get_state()[0], hp)


@pytest.mark.parametrize("graphs", [True, False])
@pytest.mark.parametrize("nsteps", [0, 1, 3])
def test_advance_matches_three_calls(BH, nsteps, graphs, monkeypatch):
    """bh_advance (velocity upload beside the first build; its first step a
    captured graph with an external event wait, or direct launches) ==
    bh_set_state + bh_step + bh_get_state, bitwise, for host and device
    buffers, with and without masses / velocities; later steps continue alike."""
    import torch

    if not graphs:
        monkeypatch.setenv("BH_NO_GRAPHS", "1")

    m, p, v = bhgen.generate("cfg2", n=5000)
    prm = bhgen.params("cfg2")
    p2 = p + np.float32(1e-3) * v  # a different state to load
    a = BH(m, p, v, **prm)
    b = BH(m, p, v, **prm)
    a.set_state(m, p2, v)
    a.step(nsteps)
    ra = a.get_state()
    rb = b.advance(m, p2, v, nsteps)
    assert np.array_equal(ra[0], rb[0]) and np.array_equal(ra[1], rb[1])
    a.step(2)
    b.step(2)
    assert all(np.array_equal(x, y) for x, y in zip(a.get_state(), b.get_state()))
    # masses kept, zero velocities
    a.set_state(None, p, None)
    a.step(nsteps)
    ra = a.get_state()
    rb = b.advance(None, p, None, nsteps)
    assert np.array_equal(ra[0], rb[0]) and np.array_equal(ra[1], rb[1])
    # device buffers
    dm, dp, dv = (torch.from_numpy(x).cuda() for x in (m, p2, v))
    po, vo = torch.empty_like(dp), torch.empty_like(dv)
    b.advance(dm, dp, dv, nsteps, po, vo)
    a.set_state(m, p2, v)
    a.step(nsteps)
    ra = a.get_state()
    assert np.array_equal(ra[0], po.cpu().numpy()) and np.array_equal(ra[1], vo.cpu().numpy())
    a.close()
    b.close()


def test_advance_multirank_matches_three_calls(BH):
    """bh_advance on a rank of a multi-rank ctx (own velocity slice, host
    scatter of the velocities) == bh_set_state + bh_step + bh_get_state."""
    m, p, v = bhgen.generate("cfg2", n=6000)
    prm = bhgen.params("cfg2")
    p2 = p + np.float32(1e-3) * v
    for r in range(2):
        a = BH(m, p, v, rank=r, world=2, **prm)
        b = BH(m, p, v, rank=r, world=2, **prm)
        b.set_state(m, p2, v)
        b.step(1)
        rb = b.get_state()
        ra = a.advance(None, p2, v, 1)
        assert np.array_equal(ra[0], rb[0]) and np.array_equal(ra[1], rb[1])
        a.close()
        b.close()


@pytest.mark.parametrize("near", ["0", "1"])
def test_sort_vs_lexsort_many_ties(BH, monkeypatch, near):
    """K2 + tie fix-up == numpy lexsort (library routine) on heavy ties, over
    several steps (ties recur in storage order != user order), on the full
    radix path and on the near-sorted path."""
    monkeypatch.setenv("BH_NEAR_SORT" if near == "1" else "BH_NO_NEAR_SORT", "1")
    rng = np.random.default_rng(9)
    pos = rng.integers(0, 16, size=(50000, 3)).astype(np.float32)
    vel = rng.normal(size=(50000, 3)).astype(np.float32)
    m = np.ones(50000, np.float32)
    bh = BH(m, pos, vel, theta=0.5, eps=0.5, dt=1e-9)
    for step in range(3):
        bh.build_tree()
        k, perm = bh.get_keys()
        gpos, _ = bh.get_state()
        o = oracle.Oracle(m, gpos.astype(np.float64), None, theta=0.5, eps=0.5).build()
        ok, operm = o.keys()
        assert np.array_equal(k, ok) and np.array_equal(perm.astype(np.int64), operm)
        user_keys = np.empty_like(ok)
        user_keys[operm] = ok
        assert np.array_equal(operm, np.lexsort((np.arange(50000), user_keys)))
        bh.step(1)


def test_step_graph_matches_direct_launches(BH, monkeypatch):
    """bh_step replays a captured CUDA graph per kick value; the direct-launch
    path (BH_NO_GRAPHS) gives bitwise the same trajectory."""
    m, p, v = bhgen.generate("cfg2", n=20000)
    prm = bhgen.params("cfg2")
    g = BH(m, p, v, **prm)
    g.step(4)
    monkeypatch.setenv("BH_NO_GRAPHS", "1")
    d = BH(m, p, v, **prm)
    d.step(4)
    gp, gv = g.get_state()
    dp, dv = d.get_state()
    assert np.array_equal(gp, dp) and np.array_equal(gv, dv)
    # graphs also survive a state reload (step counter reset -> half-kick graph)
    g.set_state(m, p, v)
    d.set_state(m, p, v)
    g.step(2)
    d.step(2)
    assert np.array_equal(g.get_state()[0], d.get_state()[0])


@pytest.mark.parametrize("hook", [{"BH_RESUME_CAP": "4"}, {"BH_RESUME_STACK": "40"}])
def test_resume_rare_paths(BH, monkeypatch, hook):
    """Targets whose fp32 MAC test was inconclusive continue in k_walk_resume.
    Its rare paths, forced by test hooks: queue slots beyond the resume-state
    capacity restart from the root; a full segment stack hands the target to
    one lane's stackless walk.  Both must still give the oracle's counts and
    forces."""
    for k, v in hook.items():
        monkeypatch.setenv(k, v)
    m, p, v = bhgen.generate("cfg3", n=300000)
    prm = bhgen.params("cfg3")
    bh = BH(m, p, v, **prm)
    bh.build_tree()
    o = _oracle(m, p, v, prm)
    check_step0(bh, o, m.shape[0])
    st = bh.get_stats()
    assert st["redo_targets"] > 4, "the input must exercise the resume path"


def test_near_sorted_path_matches_full_sort(BH, monkeypatch):
    """The near-sorted sort (keys in the previous build's order, out-of-order
    keys sorted apart and merged) gives bitwise the full radix sort's keys,
    permutation and trajectory, and falls back to the full sort when the
    order is lost (positions permuted by set_state)."""
    m, p, v = bhgen.generate("cfg2", n=50000)
    prm = bhgen.params("cfg2")
    monkeypatch.setenv("BH_NEAR_SORT", "1")  # on below its automatic size threshold too
    a = BH(m, p, v, **prm)
    monkeypatch.delenv("BH_NEAR_SORT")
    monkeypatch.setenv("BH_NO_NEAR_SORT", "1")
    b = BH(m, p, v, **prm)
    monkeypatch.delenv("BH_NO_NEAR_SORT")
    for _ in range(3):
        a.step(1)
        b.step(1)
        a.build_tree()
        b.build_tree()
        ka, pa = a.get_keys()
        kb, pb = b.get_keys()
        assert np.array_equal(ka, kb) and np.array_equal(pa, pb)
        assert a.get_stats()["near_sorted"] == 1 and b.get_stats()["near_sorted"] == 0
    assert np.array_equal(a.get_state()[0], b.get_state()[0])
    # a scrambled state: the previous order is useless -> full sort, same result
    rng = np.random.default_rng(3)
    perm = rng.permutation(m.shape[0])
    a.set_state(m, p[perm], v[perm])
    b.set_state(m, p[perm], v[perm])
    a.build_tree()
    b.build_tree()
    assert a.get_stats()["near_sorted"] == 0
    ka, pa = a.get_keys()
    kb, pb = b.get_keys()
    assert np.array_equal(ka, kb) and np.array_equal(pa, pb)
    o = _oracle(m, p[perm], v[perm], prm)
    ok, operm = o.keys()
    assert np.array_equal(ka, ok) and np.array_equal(pa.astype(np.int64), operm)


@pytest.mark.parametrize("world", [2, 3])
def test_partition_cost_split_bitwise(BH, world):
    """Equal-cost ownership (bh_set_partition with bounds from the last walk's
    interaction counts, dist.cost_bounds): every rank's forces, positions and
    velocities after a step are bitwise the P = 1 ones; the velocities handed
    over survive the move."""
    from paper_1109_5190_b200 import dist as bdist

    m, p, v = bhgen.generate("cfg2", n=30000)
    prm = bhgen.params("cfg2")
    one = BH(m, p, v, **prm)
    one.build_tree()
    ref = one.compute_forces()
    costs, vel_all = one.get_own()  # P = 1: every particle, storage order
    _, perm = one.get_keys()        # storage order == step-0 Morton order
    one.step(1)
    ref_pos, ref_vel = one.get_state()
    bounds = bdist.cost_bounds(costs, world)
    assert bounds != [len(m) * r // world for r in range(world + 1)]  # a real move
    got = np.full_like(ref, np.nan)
    got_pos = np.full_like(ref, np.nan)
    got_vel = np.full_like(ref, np.nan)
    for r in range(world):
        bh = BH(m, p, v, rank=r, world=world, **prm)
        bh.set_partition(bounds, vel_all[bounds[r]:bounds[r + 1]])
        st = bh.get_stats()
        assert (st["own_begin"], st["own_end"]) == (bounds[r], bounds[r + 1])
        assert np.array_equal(bh.get_own()[1], vel_all[bounds[r]:bounds[r + 1]])
        own = perm[bounds[r]:bounds[r + 1]].astype(np.int64)
        bh.build_tree()
        a = bh.compute_forces()
        got[own] = a[own]
        bh.step(1)
        pos, vel = bh.get_state()
        got_pos[own] = pos[own]
        got_vel[own] = vel[own]
    assert not np.isnan(got).any()
    assert np.array_equal(got, ref)
    assert np.array_equal(got_pos, ref_pos) and np.array_equal(got_vel, ref_vel)
    # and the partitioned result against the oracle: counts exact, forces and
    # the one-step state within 1e-4
    o = _oracle(m, p, v, prm)
    oacc, ocnt = o.forces()
    assert np.array_equal(costs.astype(np.int64)[np.argsort(perm)], ocnt)  # storage -> user order
    assert relerr(got, oacc).max() < TOL
    o.step(1)
    opos, ovel = o.state()
    assert relerr(got_pos, opos).max() < TOL and relerr(got_vel, ovel).max() < TOL


@pytest.mark.parametrize("world,rebalance_at", [(2, None), (3, 2)])
def test_multirank_steps_external_exchange_bitwise(BH, world, rebalance_at):
    """The multi-GPU step loop with P single-GPU ranks in one process: each rank
    builds the full tree, walks and integrates its own range; the exchange of
    K8 is done by the caller (bh_get_pos4 / bh_set_pos4: every owner's slice to
    every rank) instead of NCCL.  After 4 steps -- with an equal-cost
    repartition in between for P = 3 -- every particle's position and velocity
    is bitwise the P = 1 trajectory."""
    from paper_1109_5190_b200 import dist as bdist

    m, p, v = bhgen.generate("cfg2", n=20000)
    prm = bhgen.params("cfg2")
    n = m.shape[0]
    one = BH(m, p, v, **prm)
    one.build_tree()
    _, perm = one.get_keys()  # step 0: storage id -> user index (storage order = step-0 Morton order)
    one.step(4)
    ref_pos, ref_vel = one.get_state()
    ranks = [BH(m, p, v, rank=r, world=world, **prm) for r in range(world)]
    bounds = [n * r // world for r in range(world + 1)]
    for k in range(4):
        if rebalance_at is not None and k == rebalance_at:
            costs = np.concatenate([bh.get_own()[0] for bh in ranks]).astype(np.float64)
            vels = np.concatenate([bh.get_own()[1] for bh in ranks])
            bounds = bdist.cost_bounds(costs, world)
            for r, bh in enumerate(ranks):
                bh.set_partition(bounds, vels[bounds[r]:bounds[r + 1]])
        for bh in ranks:
            bh.step(1)
        slices = [ranks[r].get_pos4(bounds[r], bounds[r + 1]) for r in range(world)]
        for q, bh in enumerate(ranks):
            for r in range(world):
                if r != q:
                    bh.set_pos4(slices[r], bounds[r], bounds[r + 1])
    got_pos = np.full_like(ref_pos, np.nan)
    got_vel = np.full_like(ref_vel, np.nan)
    for r, bh in enumerate(ranks):
        pos, vel = bh.get_state()
        own = perm[bounds[r]:bounds[r + 1]].astype(np.int64)
        got_pos[own] = pos[own]
        got_vel[own] = vel[own]
        # the replicated positions agree everywhere, not only on the own range
        assert np.array_equal(pos, ref_pos)
    assert np.array_equal(got_pos, ref_pos) and np.array_equal(got_vel, ref_vel)
    # against the free-running oracle over the same 4 steps
    o = _oracle(m, p, v, prm)
    o.step(4)
    opos, ovel = o.state()
    assert relerr(got_pos, opos).max() < TOL


@pytest.mark.parametrize("world,rebalance_at", [(2, None), (3, 2)])
def test_fused_exchange_peer_stores_bitwise(BH, world, rebalance_at):
    """K8 fused into K7 (bh_set_peers, NEXT-1): P single-GPU ranks in one
    process, each holding the others' pos4 replicas as peer pointers; every
    step is all ranks' bh_step_phase(0) (build), a sync, then all ranks'
    bh_step_phase(1) (walk + leapfrog storing each new own position into every
    replica), a sync -- no exchange call at all.  After 4 steps (an equal-cost
    repartition in between for P = 3) every replica holds bitwise the P = 1
    positions, the own velocities are bitwise P = 1's, and the trajectory is
    within 1e-4 of the free-running oracle."""
    m, p, v = bhgen.generate("cfg2", n=20000)
    prm = bhgen.params("cfg2")
    n = m.shape[0]
    one = BH(m, p, v, **prm)
    one.build_tree()
    _, perm = one.get_keys()
    one.step(4)
    ref_pos, ref_vel = one.get_state()
    from paper_1109_5190_b200 import dist as bdist

    ranks = [BH(m, p, v, rank=r, world=world, **prm) for r in range(world)]
    ptrs = [bh.pos4_ptr() for bh in ranks]
    assert len(set(ptrs)) == world
    for bh in ranks:
        bh.set_peers(ptrs)
    bounds = [n * r // world for r in range(world + 1)]
    for k in range(4):
        if rebalance_at is not None and k == rebalance_at:
            costs = np.concatenate([bh.get_own()[0] for bh in ranks]).astype(np.float64)
            vels = np.concatenate([bh.get_own()[1] for bh in ranks])
            bounds = bdist.cost_bounds(costs, world)
            for r, bh in enumerate(ranks):
                bh.set_partition(bounds, vels[bounds[r]:bounds[r + 1]])
        for bh in ranks:
            bh.step_phase(0)
        for bh in ranks:
            bh.sync()
        for bh in ranks:
            bh.step_phase(1)
        for bh in ranks:
            bh.sync()
    got_vel = np.full_like(ref_vel, np.nan)
    for r, bh in enumerate(ranks):
        pos, vel = bh.get_state()
        assert np.array_equal(pos, ref_pos)  # every replica, all particles
        own = perm[bounds[r]:bounds[r + 1]].astype(np.int64)
        got_vel[own] = vel[own]
    assert np.array_equal(got_vel, ref_vel)
    with pytest.raises(Exception):
        ranks[0].step_phase(1)  # phase 1 needs a fresh phase 0
    with pytest.raises(Exception):
        ranks[0].step(1)  # peers without a communicator: only bh_step_phase orders the ranks
    for bh in ranks:
        bh.set_peers(None)
    o = _oracle(m, p, v, prm)
    o.step(4)
    opos, ovel = o.state()
    assert relerr(ref_pos, opos).max() < TOL and relerr(got_vel, ovel).max() < TOL


@pytest.mark.parametrize("cfg,n", [("cfg2", 30000), ("cfg3", 40000)])
def test_quadrupole_parity(BH, cfg, n):
    """multipole = 2 (NEXT-3, reading L25): keys / tree / fp64 moments AND fp64
    quadrupoles bit-identical to the extended oracle, interaction counts equal
    (the MAC does not change), accelerations within 1e-4, two free-running
    steps within 1e-4 -- and closer to the direct sum than the monopole."""
    m, p, v = bhgen.generate(cfg, n=n)
    prm = bhgen.params(cfg)
    bh = BH(m, p, v, multipole=2, **prm)
    bh.build_tree()
    o = oracle.Oracle(m, np.asarray(p, np.float64), np.asarray(v, np.float64), multipole=2, **prm).build()
    acc, err = check_step0(bh, o, n)
    assert np.array_equal(bh.get_quadrupoles(), o.quadrupoles()), "fp64 quadrupoles not bit-identical"
    # more accurate than the monopole against the exact direct sum
    tg = np.arange(0, n, 97)
    ref = oracle.direct(m, np.asarray(p, np.float64), prm["eps"], prm["G"], targets=tg)
    mono = BH(m, p, v, **prm)
    mono.build_tree()
    am = mono.compute_forces()
    e_q = np.median(relerr(acc[tg], ref))
    e_m = np.median(relerr(am[tg], ref))
    assert e_q < 0.5 * e_m, (e_q, e_m)
    # every group size: the same counts, forces to rounding
    for g in (66, 67, 68):
        b = BH(m, p, v, multipole=2, walk_group=g, **prm)
        b.build_tree()
        assert relerr(b.compute_forces(), acc).max() < 1e-5, g
        assert np.array_equal(b.get_interactions()[0], bh.get_interactions()[0]), g
    bh.step(2)
    o.step(2)
    assert relerr(bh.get_state()[0], o.state()[0]).max() < TOL


def test_quadrupole_arg_checks(BH):
    from paper_1109_5190_b200.bh import BhError

    m, p, v = bhgen.generate("cfg1")
    with pytest.raises(BhError) as e:
        BH(m, p, v, theta=0.5, eps=1e-3, multipole=3)
    assert e.value.code == -1
    with pytest.raises(BhError) as e:
        BH(m, p, v, theta=0.5, eps=1e-3, multipole=2, walk_group=80)  # not a walk_group code
    assert e.value.code == -1
    b = BH(m, p, v, theta=0.5, eps=1e-3)
    b.build_tree()
    with pytest.raises(BhError):
        b.get_quadrupoles()  # monopole ctx


@pytest.mark.parametrize("multipole", [1, 2])
def test_poisoned_workspace_same_results(BH, monkeypatch, multipole):
    """Every workspace byte set to 0xFF at create (NaN as floats, huge as
    indices): a kernel that read memory nothing had written would change the
    results or fault.  Three steps, forces and quadrupoles must be bitwise
    those of a normal workspace."""
    m, p, v = bhgen.generate("cfg2", n=25000)
    prm = bhgen.params("cfg2")
    monkeypatch.setenv("BH_NEAR_SORT", "1")  # cover the near-sorted path too
    ref = BH(m, p, v, multipole=multipole, **prm)
    monkeypatch.setenv("BH_POISON_WORKSPACE", "1")
    got = BH(m, p, v, multipole=multipole, **prm)
    monkeypatch.delenv("BH_POISON_WORKSPACE")
    for bh in (ref, got):
        bh.step(3)
        bh.build_tree()
    assert np.array_equal(ref.compute_forces(), got.compute_forces())
    assert np.array_equal(ref.get_state()[0], got.get_state()[0])
    assert np.array_equal(ref.get_state()[1], got.get_state()[1])
    if multipole == 2:
        assert np.array_equal(ref.get_quadrupoles(), got.get_quadrupoles())


@pytest.mark.slow
@pytest.mark.skipif(not os.environ.get("BH_SLOW"), reason="BH_SLOW=1: the ~10-minute free-running cfg4 run")
def test_cfg4_free_running_full(BH):
    """cfg4 free-running on both sides for its 5 stated steps (the fp64 oracle
    steps all 2^24 particles from its own fp64 state): positions of every
    particle within 1e-4 after step 5; velocities reported.  Writes a summary
    to gpurun_out/cfg4_free_running.json (committed under profiles/)."""
    import json
    import time

    c = bhgen.CONFIGS["cfg4"]
    m, p, v = bhgen.generate("cfg4")
    prm = bhgen.params("cfg4")
    bh = BH(m, p, v, **prm)
    bh.step(c.steps)
    gpos, gvel = bh.get_state()
    t0 = time.time()
    o = oracle.Oracle(m, p.astype(np.float64), v.astype(np.float64), **prm)
    inter = o.step(c.steps)
    t_or = time.time() - t0
    opos, ovel = o.state()
    pe, ve = relerr(gpos, opos), relerr(gvel, ovel)
    out = {"config": "cfg4", "n": int(m.shape[0]), "steps": c.steps, "oracle_seconds": t_or,
           "oracle_interactions_per_step": [int(x) for x in inter],
           "pos_rel_err": {"max": float(pe.max()), "p99": float(np.quantile(pe, 0.99)), "median": float(np.median(pe))},
           "vel_rel_err": {"max": float(ve.max()), "p99": float(np.quantile(ve, 0.99)), "median": float(np.median(ve))},
           "vel_over_1e-4": int((ve >= TOL).sum())}
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/cfg4_free_running.json", "w") as f:
        json.dump(out, f, indent=1)
    print(out)
    assert pe.max() < TOL
