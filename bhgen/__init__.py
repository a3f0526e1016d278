"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NONE of the Barnes-Hut arithmetic: it only draws particles.
It is the one module both sides may import (task rule ③).  Every array it
returns is canonical fp32 (mass[N], pos[N,3], vel[N,3]); the oracle promotes
them exactly to fp64, the GPU reads them as-is, so libm differences between
languages never matter.

Generator recipe (SURVEY.md §8(d) "Generator (H1)", SPEC.md:415-424 icgen):

* splitmix64: state += 0x9E3779B97F4A7C15; z = state;
  z = (z ^ z>>30)*0xBF58476D1CE4E5B9; z = (z ^ z>>27)*0x94D049BB133111EB;
  out = z ^ z>>31.  unit = (out >> 11) * 2^-53.
* Counter-based per particle: seed_i = the i-th (0-based) output of the
  stream started at state = seed; particle i's k-th draw (0-based) is output
  k of the stream started at state = seed_i, i.e. mix(seed_i + (k+1)*golden).
  Every particle's draws are independent of N, so a prefix of a larger
  configuration equals the smaller one.
* Fixed draw order per particle:
  uniform: x, y, z, then (lognormal masses) u1, u2 (Box-Muller,
  z = sqrt(-2 ln(1-u1)) cos(2 pi u2)).
  Plummer ("standard Plummer model"; SPEC.md:424 recipe):
  repeat {u -> r = a/sqrt(u^(-2/3)-1)} until r < rcut*a; z~U[-1,1], phi~U[0,2pi)
  for the position direction; repeat {q, y} until 0.1*y < q^2 (1-q^2)^(7/2);
  z, phi for the velocity direction; speed q*v_esc, v_esc = sqrt(2)(1+r^2)^(-1/4)
  sqrt(G M / a).
* Normalisations (lognormal sum, COM / momentum shifts, per sphere for cfg5)
  in fp64, then a single rounding to fp32.

The five BASELINE.json configs are in CONFIGS (cfg1..cfg5).  The paper's own
inputs came from Piet Hut's Plummer generator, which is not
available; these seeded samples stand in for them.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_TWO_M53 = 2.0 ** -53


def _mix(z: np.ndarray) -> np.ndarray:
    """splitmix64 output function on an array of post-increment states."""
    z = np.asarray(z, dtype=np.uint64)
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def splitmix64_outputs(seed: int, count: int, start: int = 0) -> np.ndarray:
    """Outputs start..start+count-1 (0-based) of splitmix64 started at `seed`."""
    k = np.arange(start + 1, start + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return _mix(np.uint64(seed) + k * GOLDEN)


def unit_from_u64(u: np.ndarray) -> np.ndarray:
    return (u >> np.uint64(11)).astype(np.float64) * _TWO_M53


class _Streams:
    """Per-particle counter-based streams for particle indices `idx`."""

    def __init__(self, seed: int, idx: np.ndarray):
        idx = np.asarray(idx, dtype=np.uint64)
        with np.errstate(over="ignore"):
            self.base = _mix(np.uint64(seed) + (idx + np.uint64(1)) * GOLDEN)
        self.ctr = np.zeros(idx.shape[0], dtype=np.uint64)

    def draw(self, sel: np.ndarray | None = None) -> np.ndarray:
        """One unit draw for the selected particles (all if sel is None)."""
        if sel is None:
            base, ctr = self.base, self.ctr
        else:
            base, ctr = self.base[sel], self.ctr[sel]
        with np.errstate(over="ignore"):
            u = unit_from_u64(_mix(base + (ctr + np.uint64(1)) * GOLDEN))
        if sel is None:
            self.ctr += np.uint64(1)
        else:
            self.ctr[sel] += np.uint64(1)
        return u


def _uniform_cube(st: _Streams, n: int) -> np.ndarray:
    pos = np.empty((n, 3), dtype=np.float64)
    for a in range(3):
        pos[:, a] = st.draw()
    return pos


def _plummer(st: _Streams, n: int, a: float, total_mass: float, rcut: float, G: float = 1.0):
    """Plummer positions/velocities in fp64 (before the COM shift)."""
    r = np.empty(n, dtype=np.float64)
    pend = np.arange(n)
    while pend.size:
        u = st.draw(pend)
        with np.errstate(divide="ignore", invalid="ignore"):
            rr = a / np.sqrt(u ** (-2.0 / 3.0) - 1.0)
        ok = rr < rcut * a  # also rejects NaN / inf (u == 1 cannot occur, u == 0 gives r == 0)
        r[pend[ok]] = rr[ok]
        pend = pend[~ok]
    z = 2.0 * st.draw() - 1.0
    phi = 2.0 * np.pi * st.draw()
    sxy = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    pos = np.stack([r * sxy * np.cos(phi), r * sxy * np.sin(phi), r * z], axis=1)

    q = np.empty(n, dtype=np.float64)
    pend = np.arange(n)
    while pend.size:
        qq = st.draw(pend)
        yy = st.draw(pend)
        ok = 0.1 * yy < qq * qq * (1.0 - qq * qq) ** 3.5
        q[pend[ok]] = qq[ok]
        pend = pend[~ok]
    vesc = np.sqrt(2.0) * (1.0 + (r / a) ** 2) ** -0.25 * np.sqrt(G * total_mass / a)
    speed = q * vesc
    z = 2.0 * st.draw() - 1.0
    phi = 2.0 * np.pi * st.draw()
    sxy = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    vel = np.stack([speed * sxy * np.cos(phi), speed * sxy * np.sin(phi), speed * z], axis=1)
    return pos, vel


def _com_shift(mass: np.ndarray, pos: np.ndarray, vel: np.ndarray):
    msum = mass.sum()
    pos = pos - (mass[:, None] * pos).sum(axis=0) / msum
    vel = vel - (mass[:, None] * vel).sum(axis=0) / msum
    return pos, vel


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    kind: str  # "uniform" | "uniform_lognormal" | "plummer" | "two_plummer"
    theta: float
    eps: float
    dt: float
    steps: int
    G: float = 1.0
    seed: int = 1
    extra: dict = field(default_factory=dict)

    def with_n(self, n: int) -> "Config":
        return Config(self.name + f"@n{n}", n, self.kind, self.theta, self.eps, self.dt,
                      self.steps, self.G, self.seed, dict(self.extra))


# BASELINE.json configs[0..4]; seed 1 for all.
CONFIGS = {
    "cfg1": Config("cfg1", 4096, "uniform", 0.5, 1e-3, 1e-3, 1),
    "cfg2": Config("cfg2", 65536, "plummer", 0.5, 1e-2, 1e-3, 10),
    "cfg3": Config("cfg3", 1 << 20, "uniform_lognormal", 0.7, 1e-3, 1e-4, 5),
    "cfg4": Config("cfg4", 1 << 24, "plummer", 0.5, 1e-3, 1e-4, 5),
    "cfg5": Config("cfg5", 1 << 26, "two_plummer", 0.7, 1e-3, 1e-4, 10),
}


def generate(cfg: Config | str, n: int | None = None):
    """Return (mass f32[N], pos f32[N,3], vel f32[N,3]) for a config.

    `n` overrides the particle count (same recipe, a smaller or larger sample);
    for two_plummer the first half of the particles is sphere A.
    """
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    n = cfg.n if n is None else int(n)
    if n < 1:
        raise ValueError("n must be >= 1")
    st = _Streams(cfg.seed, np.arange(n))
    if cfg.kind == "uniform":
        pos = _uniform_cube(st, n)
        vel = np.zeros((n, 3))
        mass = np.full(n, 1.0 / n)
    elif cfg.kind == "uniform_lognormal":
        pos = _uniform_cube(st, n)
        u1 = st.draw()
        u2 = st.draw()
        zn = np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * np.pi * u2)
        w = np.exp(0.5 * zn)  # lognormal(mu=0, sigma=0.5)
        mass = w / w.sum()
        vel = np.zeros((n, 3))
    elif cfg.kind == "plummer":
        pos, vel = _plummer(st, n, 1.0, 1.0, 10.0, cfg.G)
        mass = np.full(n, 1.0 / n)
        pos, vel = _com_shift(mass, pos, vel)
    elif cfg.kind == "two_plummer":
        half = n // 2
        pos, vel = _plummer(st, n, 1.0, 0.5, 10.0, cfg.G)
        mass = np.full(n, 1.0 / n)
        for sl, sign in ((slice(0, half), 1.0), (slice(half, n), -1.0)):
            if sl.stop - (sl.start or 0) <= 0:
                continue
            p, v = _com_shift(mass[sl], pos[sl], vel[sl])
            pos[sl] = p + sign * np.array([4.0, 0.0, 0.0])
            vel[sl] = v - sign * np.array([0.3, 0.1, 0.0])
    else:
        raise ValueError(cfg.kind)
    return (mass.astype(np.float32), np.ascontiguousarray(pos, dtype=np.float32),
            np.ascontiguousarray(vel, dtype=np.float32))


def digest(mass: np.ndarray, pos: np.ndarray, vel: np.ndarray) -> str:
    h = hashlib.sha256()
    for a in (mass, pos, vel):
        h.update(np.ascontiguousarray(a, dtype=np.float32).tobytes())
    return h.hexdigest()


def params(cfg: Config | str) -> dict:
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    return dict(theta=cfg.theta, eps=cfg.eps, G=cfg.G, dt=cfg.dt)
