"""Pins of the seeded input generators (bhgen): SPEC.md:415-444 icgen, the
BASELINE.json config recipes and SURVEY.md §8(d) H1."""
import numpy as np

import bhgen


def test_splitmix64_reference_values():
    # SPEC.md:416 "seed 0 -> first u64 = 0xE220A8397B1DCDAF"
    assert int(bhgen.splitmix64_outputs(0, 1)[0]) == 0xE220A8397B1DCDAF
    # seed 1 first output 0x910A2DEC89025CC1
    assert int(bhgen.splitmix64_outputs(1, 1)[0]) == 0x910A2DEC89025CC1
    # stream continuation: outputs k..k+n of one call equal the slice of a longer call
    a = bhgen.splitmix64_outputs(7, 100)
    b = bhgen.splitmix64_outputs(7, 10, start=50)
    assert np.array_equal(a[50:60], b)


def _sm64_scalar(state):
    state = (state + 0x9E3779B97F4A7C15) & (2 ** 64 - 1)
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2 ** 64 - 1)
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2 ** 64 - 1)
    return state, z ^ (z >> 31)


def test_splitmix64_matches_sequential_definition():
    """The vectorised counter form equals the sequential SPEC.md:416 recurrence."""
    st = 12345
    seq = []
    for _ in range(20):
        st, out = _sm64_scalar(st)
        seq.append(out)
    assert [int(x) for x in bhgen.splitmix64_outputs(12345, 20)] == seq


def test_units_and_determinism_and_prefix():
    m1, p1, v1 = bhgen.generate("cfg2", n=3000)
    m2, p2, v2 = bhgen.generate("cfg2", n=3000)
    assert bhgen.digest(m1, p1, v1) == bhgen.digest(m2, p2, v2)
    _, pu, _ = bhgen.generate("cfg1")
    assert pu.min() >= 0 and pu.max() < 1 and pu.dtype == np.float32
    # uniform positions are per-particle streams: a prefix of a larger N is identical
    _, pbig, _ = bhgen.generate("cfg1", n=8192)
    assert np.array_equal(pbig[:4096], pu)


def test_cfg1_cfg3_recipes():
    m, p, v = bhgen.generate("cfg1")
    assert m.shape == (4096,) and np.all(m == np.float32(1 / 4096)) and np.all(v == 0)
    m, p, v = bhgen.generate("cfg3", n=1 << 16)
    w = np.log(m.astype(np.float64))
    assert abs(w.std() - 0.5) < 0.01            # lognormal sigma 0.5
    assert abs(m.astype(np.float64).sum() - 1) < 1e-5 and np.all(v == 0)


def test_plummer_profile_truncated():
    """Plummer, truncated at 10a: M(<a)/M = 0.3589 and the
    half-mass radius 1.2875a (analytic M(r) = r^3/(1+r^2)^1.5
    renormalised by M(10a))."""
    m, p, v = bhgen.generate("cfg2")
    r = np.linalg.norm(p.astype(np.float64), axis=1)
    assert abs(np.mean(r < 1.0) - 0.3589) < 0.01
    assert abs(np.median(r) - 1.2875) / 1.2875 < 0.03
    assert r.max() < 10.5
    # analytic check of the two constants themselves
    Mr = lambda x: x ** 3 / (1 + x * x) ** 1.5
    assert abs(Mr(1.0) / Mr(10.0) - 0.3589) < 1e-4
    assert abs(Mr(1.2875) / Mr(10.0) - 0.5) < 1e-3
    # COM frame and unit total mass (fp64 before rounding: checked to fp32 level)
    m64 = m.astype(np.float64)
    assert abs(m64.sum() - 1) < 1e-6
    assert np.linalg.norm((m64[:, None] * p).sum(0)) < 1e-6
    assert np.linalg.norm((m64[:, None] * v).sum(0)) < 1e-6


def test_plummer_virial_equilibrium():
    """Velocities from the Plummer distribution function: 2K/|W| ~ 1."""
    m, p, v = bhgen.generate("cfg2", n=4096)
    m64, x, u = m.astype(np.float64), p.astype(np.float64), v.astype(np.float64)
    K = 0.5 * (m64 * (u * u).sum(1)).sum()
    W = 0.0
    for i in range(len(m64)):
        d = x[i + 1:] - x[i]
        W -= (m64[i] * m64[i + 1:] / np.sqrt((d * d).sum(1))).sum()
    assert abs(2 * K / abs(W) - 1.0) < 0.1


def test_two_plummer_recipe():
    n = 1 << 14
    m, p, v = bhgen.generate("cfg5", n=n)
    a, b = p[: n // 2].astype(np.float64), p[n // 2:].astype(np.float64)
    m64 = m.astype(np.float64)
    assert abs(m64[: n // 2].sum() - 0.5) < 1e-6
    np.testing.assert_allclose(a.mean(0), [4, 0, 0], atol=0.1)
    np.testing.assert_allclose(b.mean(0), [-4, 0, 0], atol=0.1)
    np.testing.assert_allclose(v[: n // 2].astype(np.float64).mean(0), [-0.3, -0.1, 0], atol=1e-5)
    np.testing.assert_allclose(v[n // 2:].astype(np.float64).mean(0), [0.3, 0.1, 0], atol=1e-5)
