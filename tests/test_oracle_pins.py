"""Pins of the fp64 CPU oracle against things other than itself (task rule ③).

Each test names the passage it follows.  Sources of truth used here:
closed forms (two-body, constant acceleration, Kepler orbit), brute force on
tiny inputs (tests/bruteforce.py: prefix enumeration, ancestor enumeration,
numpy direct sum), library routines (numpy lexsort), the worked example of
tests/golden/ and invariants (momentum, energy, theta monotonicity).
"""
import json
import math
import os

import numpy as np
import pytest

import bhgen
import oracle
from tests import bruteforce as bf

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _orc(mass, pos, vel=None, **kw):
    return oracle.Oracle(np.asarray(mass, np.float64), np.asarray(pos, np.float64), vel, **kw)


# ----------------------------------------------------------------- keys / cube
def test_worked_example_keys_tree_forces():
    """SURVEY.md §8(c) worked example == SPEC.md:175, analogue of PAPER.md Fig. 2
    (lines 457-466: P1 'requires only two inputs')."""
    g = _gold("worked_example.json")
    P = np.array(g["positions"], np.float32)
    for theta in (0.3, 0.5, 0.7):
        o = _orc(g["masses"], P.astype(np.float64), theta=theta, eps=g["eps"]).build()
        lo, L, _ = o.root()
        assert list(lo) == g["lo"] and L == np.float32(g["L_float32"])
        k, perm = o.keys()
        assert [hex(int(x)) for x in k] == g["keys_hex"]
        assert list(perm) == g["perm"]
        lv, fi, co = o.tree()
        assert [list(map(int, t)) for t in zip(lv, fi, co)] == g["dfs_nodes_level_first_count"]
        a, c = o.forces()
        assert list(c) == g["counts_theta_0.3_to_0.7"]
        np.testing.assert_allclose(a[0], g["a_P1_theta_0.3_to_0.7"], atol=1e-8)
        # closed form on the fp32 inputs: P2 (mass 1) + centroid of P3, P4 (mass 2)
        X = P.astype(np.float64)
        cen = (X[2] + X[3]) / 2
        cf = (X[1] - X[0]) / np.linalg.norm(X[1] - X[0]) ** 3 + 2 * (cen - X[0]) / np.linalg.norm(cen - X[0]) ** 3
        np.testing.assert_allclose(a[0], cf, rtol=1e-14)
    o = _orc(g["masses"], P.astype(np.float64), theta=0.0, eps=0.0).build()
    a, c = o.forces()
    assert list(c) == g["counts_theta_0"]
    np.testing.assert_allclose(a[0], g["a_P1_theta_0"], atol=1e-8)
    # just below the two-input threshold P1 needs all three particles
    o = _orc(g["masses"], P.astype(np.float64), theta=0.158, eps=0.0).build()
    assert o.forces()[1][0] == 3
    o = _orc(g["masses"], P.astype(np.float64), theta=0.159, eps=0.0).build()
    assert o.forces()[1][0] == 2


def test_interleave_exhaustive_per_axis():
    """Keys are the x-major 3-bit interleave of the 21-bit cell coordinates
    (reading L10/L12).  Exhaustive over all 2^21 values per axis: positions
    x = q on an integer grid make scale exactly 1 (L = 2^21)."""
    q = np.arange(1 << 21, dtype=np.int64)
    qy = (q * 7) % (1 << 21)
    qz = (q * 13 + 5) % (1 << 21)
    pos = np.stack([q, qy, qz], axis=1).astype(np.float64)
    pos = np.vstack([pos, [[float(1 << 21)] * 3]])  # sets lo = 0, L = 2^21
    o = _orc(np.ones(pos.shape[0]), pos, theta=0.5, eps=1e-3).build()
    lo, L, scale = o.root()
    assert list(lo) == [0, 0, 0] and L == 2.0 ** 21 and scale == 1.0
    k, perm = o.keys()
    user_keys = np.empty_like(k)
    user_keys[perm] = k
    dec = bf.decode_keys_np(user_keys[:-1]).astype(np.int64)
    assert np.array_equal(dec[:, 0], q) and np.array_equal(dec[:, 1], qy) and np.array_equal(dec[:, 2], qz)
    # x = hi quantises to 2^21 and is clamped to 2^21 - 1 (reading L10)
    assert bf.decode_key(int(user_keys[-1])) == ((1 << 21) - 1,) * 3
    # spot values against the bit-by-bit definition
    for (a, b, c) in [(1, 0, 0), (0, 1, 0), (0, 0, 1), ((1 << 21) - 1, 0, 0), (5, 3, 6)]:
        assert bf.decode_key(oracle.interleave(a, b, c)) == (a, b, c)
    assert oracle.interleave(1, 0, 0) == 4 and oracle.interleave(0, 1, 0) == 2 and oracle.interleave(0, 0, 1) == 1


def test_quantisation_cells_contain_points():
    """Each particle lies in (or, by fp32 rounding, on the boundary of) the
    level-21 cell its key names; x = lo -> 0, x = hi -> 2^21-1 (L10/L11)."""
    m, p, _ = bhgen.generate("cfg2", n=4096)
    o = _orc(m, p.astype(np.float64), theta=0.5, eps=0.01).build()
    lo, L, scale = o.root()
    k, perm = o.keys()
    q = bf.decode_keys_np(k).astype(np.float64)
    x = p[perm].astype(np.float64)
    cell = float(L) / 2 ** 21
    lo64 = lo.astype(np.float64)
    # containment up to the fp32 rounding of the scaled coordinate: three
    # roundings of relative size 2^-24 on t < 2^21 -> < 0.19 cells
    t = (x - lo64) / cell
    assert np.all(t >= q - 0.25) and np.all(t <= q + 1 + 0.25)
    assert np.mean((t >= q) & (t < q + 1)) > 0.9
    mins = np.argmin(p, axis=0)
    for a in range(3):
        assert int(bf.decode_key(int(k[np.where(perm == mins[a])[0][0]]))[a]) == 0
    arg = int(np.argmax(p[:, 0] - lo[0]))
    if p[arg, 0] - lo[0] == L:
        assert bf.decode_key(int(k[np.where(perm == arg)[0][0]]))[0] == (1 << 21) - 1


def test_degenerate_cube_all_coincident():
    """L == 0 -> scale 0 -> every key 0; the tree is a 22-node chain whose last
    node is a bucket of all particles (L9, SURVEY.md §8(c) topology pin)."""
    pos = np.tile([[0.25, -3.0, 7.5]], (7, 1))
    o = _orc(np.ones(7), pos, theta=0.5, eps=0.1).build()
    _, L, scale = o.root()
    assert L == 0 and scale == 0
    k, perm = o.keys()
    assert np.all(k == 0) and list(perm) == list(range(7))
    lv, fi, co = o.tree()
    assert list(lv) == list(range(22)) and np.all(fi == 0) and np.all(co == 7)
    a, c = o.forces()
    assert np.all(c == 6) and np.all(a == 0.0)
    # eps == 0 with coincident particles is an error, not a silent inf
    o = _orc(np.ones(7), pos, theta=0.5, eps=0.0).build()
    with pytest.raises(oracle.OracleError):
        o.forces()


def test_sort_tiebreak_and_lexsort():
    """Reading L13: stable ascending sort, ties by ascending user index."""
    g = _gold("sort_tiebreak.json")
    pos = np.array([g[s] for s in g["order"]], np.float64)
    o = _orc(np.ones(5), pos, theta=0.5, eps=0.1).build()
    assert list(o.keys()[1]) == g["perm"]
    # random keys with many duplicates vs numpy's lexsort (a library routine)
    rng = np.random.default_rng(3)
    pos = rng.integers(0, 4, size=(3000, 3)).astype(np.float64)
    o = _orc(np.ones(3000), pos, theta=0.5, eps=0.1).build()
    k, perm = o.keys()
    user_keys = np.empty_like(k)
    user_keys[perm] = k
    assert np.array_equal(perm, np.lexsort((np.arange(3000), user_keys)))
    assert np.all(np.diff(k.astype(np.float64)) >= 0)


# ----------------------------------------------------------------- topology
@pytest.mark.parametrize("case", ["uniform17", "uniform1000", "plummer4096", "dups", "n1", "n2", "faces"])
def test_topology_vs_prefix_enumeration(case):
    """Octree = brute-force prefix enumeration (L9, L15, L16)."""
    rng = np.random.default_rng(11)
    if case == "uniform17":
        pos = rng.random((17, 3))
    elif case == "uniform1000":
        pos = rng.random((1000, 3))
    elif case == "plummer4096":
        _, p, _ = bhgen.generate("cfg2", n=4096)
        pos = p.astype(np.float64)
    elif case == "dups":  # 2000 uniform + 55 exact copies -> buckets of 2-3
        base = rng.random((2000, 3)).astype(np.float32).astype(np.float64)
        pos = np.vstack([base, base[rng.integers(0, 2000, 55)]])
    elif case == "n1":
        pos = np.array([[1.0, 2.0, 3.0]])
    elif case == "n2":
        pos = np.array([[0.0, 0.0, 0.0], [1e-7, 0.0, 0.0]])
    else:  # particles on the faces of the bounding box
        pos = rng.integers(0, 3, size=(300, 3)).astype(np.float64) * 0.5
    n = pos.shape[0]
    o = _orc(np.ones(n), pos, theta=0.5, eps=0.1).build()
    k, _ = o.keys()
    lv, fi, co = o.tree()
    got = [tuple(map(int, t)) for t in zip(lv, fi, co)]
    assert got == bf.prefix_nodes(k)
    # invariants: single-particle leaves + bucket members = N
    leaves = co == 1
    buckets = (lv == 21) & (co >= 2)
    assert co[leaves].sum() + co[buckets].sum() == n
    if case == "dups":
        assert buckets.sum() > 0


# ----------------------------------------------------------------- moments
def test_moments_spec_examples_and_flat_sums():
    """SPEC.md:183-185 compute_moments examples; every node's M and MX equal
    the flat sums over its particle range (L14) within 1e-12 relative."""
    o = _orc([1.0, 1.0], [[-1, 0, 0], [1, 0, 0]], theta=0.5, eps=0.0).build()
    lv, fi, co, M, MX = o.tree(with_moments=True)
    assert M[0] == 2.0 and np.all(MX[0] / M[0] == 0.0)
    o = _orc([1.0, 3.0], [[0, 0, 0], [4, 0, 0]], theta=0.5, eps=0.0).build()
    lv, fi, co, M, MX = o.tree(with_moments=True)
    assert M[0] == 4.0 and MX[0, 0] / M[0] == 3.0
    m, p, _ = bhgen.generate("cfg3", n=5000)
    o = _orc(m, p.astype(np.float64), theta=0.7, eps=1e-3).build()
    _, perm = o.keys()
    lv, fi, co, M, MX = o.tree(with_moments=True)
    m64 = m.astype(np.float64)
    p64 = p.astype(np.float64)
    for t in range(len(lv)):
        mem = perm[fi[t]:fi[t] + co[t]]
        Mf = m64[mem].sum()
        assert abs(M[t] - Mf) <= 1e-12 * Mf
        np.testing.assert_allclose(MX[t] / M[t], (m64[mem, None] * p64[mem]).sum(0) / Mf, rtol=1e-12, atol=1e-15)
        if co[t] == 1:  # leaf: exact
            assert M[t] == m64[mem[0]] and np.array_equal(MX[t], m64[mem[0]] * p64[mem[0]])


# ----------------------------------------------------------------- forces
@pytest.mark.parametrize("theta", [0.0, 0.5, 0.7])
def test_two_body_closed_form(theta):
    """unit mass at distance 2, eps = 0 -> a = (0.25, 0, 0); and
    the reading-L5 counterexample (m=0.1 at 0, m=1 at (1,1,1), theta=0.7):
    with cells containing the target force-opened the result is the closed form."""
    o = _orc([1.0, 1.0], [[0, 0, 0], [2, 0, 0]], theta=theta, eps=0.0).build()
    a, c = o.forces()
    assert np.array_equal(a[0], [0.25, 0, 0]) and np.array_equal(a[1], [-0.25, 0, 0])
    assert list(c) == [1, 1]
    o = _orc([0.1, 1.0], [[0, 0, 0], [1, 1, 1]], theta=theta, eps=0.0).build()
    a, c = o.forces()
    cf = np.ones(3) * 1.0 / 3.0 ** 1.5
    np.testing.assert_allclose(a[0], cf, rtol=1e-15)
    np.testing.assert_allclose(a[1], -0.1 * cf, rtol=1e-15)


def test_softened_pair():
    eps = 0.3
    o = _orc([2.0, 1.0], [[0, 0, 0], [0, 0.5, 0]], theta=0.5, eps=eps).build()
    a, _ = o.forces()
    np.testing.assert_allclose(a[0], [0, 1.0 * 0.5 / (0.25 + eps * eps) ** 1.5, 0], rtol=1e-15)
    o = _orc([2.0, 1.0], [[0, 0, 0], [0, 0.5, 0]], theta=0.5, eps=eps, G=6.5).build()
    np.testing.assert_allclose(o.forces()[0][0, 1], 6.5 * 0.5 / (0.25 + eps * eps) ** 1.5, rtol=1e-15)


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3"])
def test_theta0_equals_direct_sum(cfg):
    """theta = 0 never accepts a cell (L4), so BH == the O(N^2) direct sum
    (SPEC.md:221); north star: 1e-12 relative.  Direct sum in numpy."""
    m, p, _ = bhgen.generate(cfg, n=2048)
    eps = bhgen.CONFIGS[cfg].eps
    o = _orc(m, p.astype(np.float64), theta=0.0, eps=eps).build()
    a, c = o.forces()
    assert np.all(c == 2047)
    ref = bf.direct_numpy(m, p, eps)
    err = np.linalg.norm(a - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert err.max() < 1e-12
    # the oracle's own direct sum agrees too
    np.testing.assert_allclose(oracle.direct(m, p, eps), ref, rtol=1e-12, atol=0)
    # momentum: sum m_i a_i = 0 (Newton's third law) to 1e-10 relative
    ma = m.astype(np.float64)[:, None] * a
    assert np.linalg.norm(ma.sum(0)) <= 1e-10 * np.abs(ma).sum()


@pytest.mark.parametrize("case", ["uniform60", "plummer120", "dups", "theta07_tight"])
def test_walk_vs_bruteforce_bh(case):
    """Recursive walk == non-recursive ancestor enumeration (PAPER.md:408-415,
    L1-L5) on tiny N: identical interaction counts, accelerations to 1e-12."""
    rng = np.random.default_rng(5)
    theta, eps = 0.5, 1e-3
    if case == "uniform60":
        pos = rng.random((60, 3)); mass = rng.random(60) + 0.5
    elif case == "plummer120":
        mass, p, _ = bhgen.generate("cfg2", n=120); pos = p.astype(np.float64)
    elif case == "dups":
        base = rng.random((50, 3)).astype(np.float32).astype(np.float64)
        pos = np.vstack([base, base[:7], base[:3]]); mass = np.ones(60)
    else:
        pos = rng.random((80, 3)) ** 3; mass = rng.random(80); theta = 0.9
    mass = np.asarray(mass, np.float64)
    for th in (theta, 0.3, 1.2):
        o = _orc(mass, pos, theta=th, eps=eps).build()
        k, perm = o.keys()
        _, L, _ = o.root()
        a, c = o.forces()
        ab, cb = bf.bh_bruteforce(mass, pos, k, perm, float(L), th, eps)
        assert np.array_equal(c, cb)
        err = np.linalg.norm(a - ab, axis=1) / np.linalg.norm(ab, axis=1)
        assert err.max() < 1e-12


def test_theta_monotone_and_accuracy_trend():
    """SPEC.md:227 theta-monotonicity of interaction counts; SPEC.md:229/541
    median error vs the direct sum decreases as theta decreases."""
    m, p, _ = bhgen.generate("cfg2", n=4096)
    ref = bf.direct_numpy(m, p, 0.01, targets=np.arange(0, 4096, 8))
    prev_c, prev_err = None, None
    for th in (0.8, 0.5, 0.3, 0.1):
        o = _orc(m, p.astype(np.float64), theta=th, eps=0.01).build()
        a, c = o.forces()
        if prev_c is not None:
            assert np.all(c >= prev_c)
        e = np.median(np.linalg.norm(a[::8] - ref, axis=1) / np.linalg.norm(ref, axis=1))
        if prev_err is not None:
            assert e < prev_err
        prev_c, prev_err = c, e
    assert prev_err < 1e-3


def test_interactions_grow_like_log_n():
    """PAPER.md:62-63 'O(N log N) computational complexity': beyond the
    near-field transient the mean interaction count per particle is affine in
    log N (a + b log N within 10%, b > 0) while N grows 16x (SPEC.md:542 trend;
    at N = 2^10 the count is still dominated by the direct near field)."""
    ns = [1 << 12, 1 << 14, 1 << 16]
    means = []
    for n in ns:
        m, p, _ = bhgen.generate("cfg2", n=n)
        o = _orc(m, p.astype(np.float64), theta=0.5, eps=0.01).build()
        means.append(o.forces()[1].mean())
    A = np.stack([np.ones(3), np.log(ns)], axis=1)
    coef, *_ = np.linalg.lstsq(A, np.array(means), rcond=None)
    fit = A @ coef
    assert coef[1] > 0
    assert np.all(np.abs(fit - means) <= 0.1 * np.array(means))
    assert means[-1] / ns[-1] < 0.25 * means[0] / ns[0]


# ----------------------------------------------------------------- leapfrog
def test_leapfrog_first_step_closed_form():
    """L8: from rest, one step gives v_1/2 = a0 dt/2 and x1 = x0 + a0 dt^2/2."""
    m, p, _ = bhgen.generate("cfg1", n=512)
    dt = 1e-3
    o = _orc(m, p.astype(np.float64), theta=0.5, eps=1e-3, dt=dt).build()
    a0, _ = o.forces()
    o.step(1)
    x1, v = o.state()
    np.testing.assert_allclose(v, a0 * dt / 2, rtol=1e-15, atol=0)
    np.testing.assert_allclose(x1, p.astype(np.float64) + a0 * dt * dt / 2, rtol=1e-15, atol=1e-18)


def test_free_particle_and_two_steps():
    """SPEC.md:358 single particle: unchanged velocity, x += v dt per step;
    second step uses the full kick v += a dt."""
    o = _orc([1.0], [[1.0, 2.0, 3.0]], vel=np.array([[0.5, -1.0, 0.25]]), theta=0.5, eps=0.0, dt=0.125)
    o.step(3)
    x, v = o.state()
    assert np.array_equal(v[0], [0.5, -1.0, 0.25])
    np.testing.assert_allclose(x[0], [1.0 + 3 * 0.0625, 2.0 - 3 * 0.125, 3.0 + 3 * 0.03125], rtol=0, atol=1e-15)
    # two bodies, two steps: the second kick is a full dt kick
    dt = 1e-2
    o = _orc([1.0, 1.0], [[-1, 0, 0], [1, 0, 0]], theta=0.0, eps=0.0, dt=dt)
    o.step(2)
    x, v = o.state()
    a0 = 0.25
    x1 = -1 + a0 * dt * dt / 2
    a1 = 1.0 / (2 * x1) ** 2
    v1 = a0 * dt / 2 + a1 * dt
    assert abs(v[0, 0] - v1) < 1e-15 and abs(x[0, 0] - (x1 + v1 * dt)) < 1e-15


@pytest.mark.slow
def test_two_body_circular_orbit():
    """m1 = m2 = 0.5, separation 1, eps = 0, theta = 0: the
    separation drifts < 1% over one period at dt = 1e-3 (Kepler closed form)."""
    dt = 1e-3
    period = 2 * math.pi  # omega^2 = G (m1 + m2) / d^3 = 1
    o = _orc([0.5, 0.5], [[-0.5, 0, 0], [0.5, 0, 0]], vel=np.array([[0, -0.5, 0], [0, 0.5, 0]]),
             theta=0.0, eps=0.0, dt=dt)
    steps = int(round(period / dt))
    worst = 0.0
    for _ in range(10):
        o.step(steps // 10)
        x, _ = o.state()
        worst = max(worst, abs(np.linalg.norm(x[1] - x[0]) - 1.0))
    assert worst < 0.01
    x, _ = o.state()
    assert np.linalg.norm(x[0] - [-0.5, 0, 0]) < 0.02  # back near the start after a period


def _energy(m, x, v, eps):
    ke = 0.5 * (m * (v * v).sum(1)).sum()
    pe = 0.0
    for i in range(len(m)):
        d = x[i + 1:] - x[i]
        pe -= (m[i] * m[i + 1:] / np.sqrt((d * d).sum(1) + eps * eps)).sum()
    return ke + pe


def test_energy_drift_theta0():
    """N = 256, theta = 0, dt = 1e-3, 100 steps: relative energy
    drift < 1e-3 (velocities synchronised with the closing half kick)."""
    m, p, v = bhgen.generate("cfg2", n=256)
    m64, eps, dt = m.astype(np.float64), 0.01, 1e-3
    e0 = _energy(m64, p.astype(np.float64), v.astype(np.float64), eps)
    o = _orc(m64, p.astype(np.float64), vel=v.astype(np.float64), theta=0.0, eps=eps, dt=dt)
    o.step(100)
    x, vh = o.state()
    o.build()
    a, _ = o.forces()
    e1 = _energy(m64, x, vh + a * dt / 2, eps)
    assert abs(e1 - e0) / abs(e0) < 1e-3
    assert abs(e0) > 0.1  # a bound system (Plummer: E ~ -0.19 in these units)


# ---------------------------------------------------------------- quadrupoles
# (multipole = 2: SURVEY.md §8(f) NEXT-3, "incorporating
# multipole moments"; reading L25 of DESIGN.md §3)

def test_quadrupole_two_masses_closed_form():
    """m1 = 1 at x = 0, m2 = 3 at x = 1: com 0.75, offsets -0.75 and 0.25;
    Q = sum m (3 y y - |y|^2 I) = diag(1.5, -0.75, -0.75) exactly."""
    m = np.array([1.0, 3.0])
    p = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0]])
    o = oracle.Oracle(m, p, theta=0.5, eps=0.0, multipole=2).build()
    Q = o.quadrupoles()
    assert np.array_equal(Q[0], [1.5, -0.75, -0.75, 0.0, 0.0, 0.0])
    lv, fi, co = o.tree()
    assert np.all(Q[co == 1] == 0.0)  # particles: no quadrupole about themselves


def test_quadrupole_parallel_axis_equals_flat_sum():
    """Every node's Q (combined bottom-up in child order) equals the flat sum
    over its particles about its centre of mass; traceless; leaves zero."""
    rng = np.random.default_rng(11)
    n = 3000
    m = rng.uniform(0.5, 2.0, n)
    p = rng.standard_normal((n, 3)) * [1.0, 0.5, 2.0]
    o = oracle.Oracle(m, p, theta=0.5, eps=0.01, multipole=2).build()
    lv, fi, co, M, MX = o.tree(with_moments=True)
    Q = o.quadrupoles()
    _, perm = o.keys()
    ps = p.astype(np.float64)[perm]  # sorted order (the oracle's fp64 state of fp32? no: fp64 input)
    ms = m[perm]
    for k in rng.choice(len(lv), 400, replace=False):
        sl = slice(fi[k], fi[k] + co[k])
        com = MX[k] / M[k]
        y = ps[sl] - com
        r2 = (y * y).sum(1)
        flat = np.array([(ms[sl] * (3 * y[:, 0] * y[:, 0] - r2)).sum(), (ms[sl] * (3 * y[:, 1] * y[:, 1] - r2)).sum(),
                         (ms[sl] * (3 * y[:, 2] * y[:, 2] - r2)).sum(), (ms[sl] * 3 * y[:, 0] * y[:, 1]).sum(),
                         (ms[sl] * 3 * y[:, 0] * y[:, 2]).sum(), (ms[sl] * 3 * y[:, 1] * y[:, 2]).sum()])
        scale = (ms[sl] * r2).sum() + 1e-300
        assert np.abs(Q[k] - flat).max() <= 1e-12 * scale + 1e-300
        assert abs(Q[k][0] + Q[k][1] + Q[k][2]) <= 1e-12 * scale + 1e-300


def _cluster_and_target(dist, seed=3):
    rng = np.random.default_rng(seed)
    a = 1.0
    cl = rng.uniform(0.0, a, (6, 3))
    mc = rng.uniform(0.5, 2.0, 6)
    tgt = np.array([[1.0, 1.0, 1.0]]) / np.sqrt(3.0) * dist + 0.5 * a
    return np.concatenate([mc, [1.0]]), np.concatenate([cl, tgt])


@pytest.mark.parametrize("order,expect", [(1, 4.0), (2, 8.0)])
def test_cell_field_convergence_order(order, expect):
    """A compact cluster seen as one cell from a far target: the relative error
    of the target's acceleration against the exact (direct) sum falls like
    (a/d)^2 for the monopole and (a/d)^3 with the quadrupole -- a wrong sign or
    factor in the quadrupole field breaks the cubic rate."""
    errs = []
    for d in (16.0, 32.0, 64.0):
        m, p = _cluster_and_target(d)
        o = oracle.Oracle(m, p, theta=0.9, eps=0.0, multipole=order).build()
        acc, cnt = o.forces(np.array([6]))
        assert cnt[0] == 1  # the cluster is one accepted cell
        ref = oracle.direct(m, p, 0.0, targets=np.array([6]))
        errs.append(np.linalg.norm(acc[0] - ref[0]) / np.linalg.norm(ref[0]))
    r1, r2 = errs[0] / errs[1], errs[1] / errs[2]
    assert 0.75 * expect < r1 < 1.3 * expect and 0.75 * expect < r2 < 1.3 * expect, (errs, r1, r2)
    if order == 2:
        m, p = _cluster_and_target(16.0)
        mono = oracle.Oracle(m, p, theta=0.9, eps=0.0).build().forces(np.array([6]))[0][0]
        quad = oracle.Oracle(m, p, theta=0.9, eps=0.0, multipole=2).build().forces(np.array([6]))[0][0]
        ref = oracle.direct(m, p, 0.0, targets=np.array([6]))[0]
        assert np.linalg.norm(quad - ref) < 0.2 * np.linalg.norm(mono - ref)


def test_quadrupole_theta0_is_direct_and_counts_unchanged():
    """theta = 0 accepts no cell: quadrupole mode is the direct sum; at any
    theta the interaction counts (the MAC decisions) do not depend on the order."""
    m, p, v = bhgen.generate("cfg1")
    pd = p.astype(np.float64)
    o2 = oracle.Oracle(m, pd, theta=0.0, eps=1e-3, multipole=2).build()
    a2, _ = o2.forces(np.arange(0, 4096, 97))
    ref = oracle.direct(m, pd, 1e-3, targets=np.arange(0, 4096, 97))
    assert np.abs(a2 - ref).max() <= 1e-12 * np.abs(ref).max()
    c1 = oracle.Oracle(m, pd, theta=0.5, eps=1e-3).build().forces()[1]
    c2 = oracle.Oracle(m, pd, theta=0.5, eps=1e-3, multipole=2).build().forces()[1]
    assert np.array_equal(c1, c2)


@pytest.mark.parametrize("eps_over_d", [0.05, 0.3, 1.0])
@pytest.mark.parametrize("G", [1.0, 2.5])
def test_softened_cell_field_is_minus_grad_potential(eps_over_d, G):
    """Reading L25 at eps > 0: an accepted cell's field is -grad of the softened
    potential Phi(x) = -G [M / r_e + (1/2) r^T Q r / r_e^5],  r = x - com,
    r_e^2 = |r|^2 + eps^2 (the monopole + quadrupole terms of the Plummer-
    softened cell, PAPER.md:755-757 future work "multipole moments").  The
    potential is evaluated here from its definition (M, com, Q summed from the
    particles in this test), differentiated by central differences, and
    compared with the oracle's contribute_cell for a target that accepts the
    cluster as one cell.  A wrong eps placement (r instead of r_e in inv5 /
    inv7), a wrong factor or sign fails at eps ~ d (the quadrupole term is
    ~1e-3 of the monopole's here, the tolerance 1e-9 of |a|)."""
    rng = np.random.default_rng(5)
    cl = rng.uniform(0.0, 1.0, (6, 3))
    mc = rng.uniform(0.5, 2.0, 6)
    d = 12.0
    tgt = 0.5 + np.array([1.0, 0.7, 0.4]) / np.linalg.norm([1.0, 0.7, 0.4]) * d
    m = np.concatenate([mc, [1.0]])
    p = np.concatenate([cl, [tgt]])
    eps = eps_over_d * d
    o2 = oracle.Oracle(m, p, theta=0.9, eps=eps, G=G, multipole=2).build()
    acc, cnt = o2.forces(np.array([6]))
    assert cnt[0] == 1  # the cluster is one accepted cell
    # the cell's moments from the particles (not from the oracle)
    M = mc.sum()
    com = (mc[:, None] * cl).sum(0) / M
    y = cl - com
    Q = np.einsum("k,ki,kj->ij", mc, 3.0 * y, y) - np.eye(3) * (mc * (y * y).sum(1)).sum()

    def phi(x):
        r = x - com
        re2 = r @ r + eps * eps
        return -G * (M / np.sqrt(re2) + 0.5 * (r @ Q @ r) / re2 ** 2.5)

    def grad(f, x, h=1e-3):  # fourth-order central differences
        return np.array([(8 * (f(x + h * e) - f(x - h * e)) - (f(x + 2 * h * e) - f(x - 2 * h * e))) / (12 * h)
                         for e in np.eye(3)])

    ref = -grad(phi, tgt)
    assert np.linalg.norm(acc[0] - ref) <= 1e-9 * np.linalg.norm(ref), (acc[0], ref)
    # and the quadrupole part alone (oracle multipole 2 minus multipole 1) against
    # -grad of the quadrupole term: it is not lost under the monopole's size
    a1, _ = oracle.Oracle(m, p, theta=0.9, eps=eps, G=G).build().forces(np.array([6]))

    def phiq(x):
        r = x - com
        re2 = r @ r + eps * eps
        return -G * 0.5 * (r @ Q @ r) / re2 ** 2.5

    gq = -grad(phiq, tgt)
    assert np.linalg.norm((acc[0] - a1[0]) - gq) <= 1e-6 * np.linalg.norm(gq), (acc[0] - a1[0], gq)


def test_step_targets_equals_full_step():
    """oracle_step_targets (the teacher-forced check of the large configs) is the
    pinned leapfrog of oracle_step restricted to the targets: bitwise equal at
    k = 0 (half kick) and k = 1 (full kick), and the state is not advanced."""
    m, p, v = bhgen.generate("cfg2", n=3000)
    prm = bhgen.params("cfg2")
    tg = np.array([0, 5, 17, 999, 2999])
    for k0 in (0, 1):
        o = oracle.Oracle(m, p.astype(np.float64), v.astype(np.float64), k0=k0, **prm)
        po, vo, cnt = o.step_targets(tg)
        p0, v0 = o.state()
        assert np.array_equal(p0, p.astype(np.float64))  # not advanced
        o.step(1)
        p1, v1 = o.state()
        assert np.array_equal(po, p1[tg]) and np.array_equal(vo, v1[tg])
        o2 = oracle.Oracle(m, p.astype(np.float64), v.astype(np.float64), k0=k0, **prm).build()
        assert np.array_equal(cnt, o2.forces(tg)[1])
