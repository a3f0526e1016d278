"""ctypes front-end of the plain fp64 CPU oracle (oracle/bh_oracle.c).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs are the only callers.  The product path
(paper_1109_5190_b200) never imports this package, and this package never
imports the product path.

Parity status of every oracle function (DESIGN.md §4 lists the pins):
  keys / root cube  -- pinned (worked example, exhaustive interleave, decode)
  sort              -- pinned (tie-break example, numpy lexsort)
  tree              -- pinned (brute-force prefix enumeration, worked example)
  moments           -- pinned (SPEC examples, flat weighted mean)
  forces / MAC      -- pinned (two-body closed form, theta=0 direct sum,
                       brute-force ancestor enumeration, worked example)
  leapfrog          -- pinned (constant-acceleration closed form, Kepler orbit,
                       energy drift)
  direct sum        -- pinned (closed forms, Newton's third law)
  quadrupoles       -- pinned (closed form of two masses, flat sum about the
                       com, tracelessness; third-order convergence of the
                       cell field against exact two-body forces)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bh_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OR_OK, OR_ERR_ARG, OR_ERR_OOM, OR_ERR_NONFINITE = 0, -1, -3, -5


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (fp-contract off: plain IEEE ops)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC",
               "-shared", "-std=c11", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        vp, i64, f64 = C.c_void_p, C.c_int64, C.c_double
        L.oracle_create.restype = vp
        L.oracle_create.argtypes = [i64, vp, vp, vp, f64, f64, f64, f64, i64]
        L.oracle_destroy.argtypes = [vp]
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_last_error.argtypes = [vp]
        L.oracle_build.argtypes = [vp]
        L.oracle_root.argtypes = [vp, vp, vp, vp]
        L.oracle_get_keys.argtypes = [vp, vp, vp]
        L.oracle_get_tree.restype = i64
        L.oracle_get_tree.argtypes = [vp, vp, vp, vp, vp, vp, i64]
        L.oracle_forces.argtypes = [vp, i64, vp, vp, vp]
        L.oracle_step.argtypes = [vp, i64, vp]
        L.oracle_get_state.argtypes = [vp, vp, vp]
        L.oracle_step_targets.argtypes = [vp, i64, vp, vp, vp, vp]
        L.oracle_direct.argtypes = [i64, vp, vp, f64, f64, i64, vp, vp]
        L.oracle_set_multipole.argtypes = [vp, C.c_int]
        L.oracle_get_quadrupoles.restype = i64
        L.oracle_get_quadrupoles.argtypes = [vp, vp, i64]
        L.oracle_interleave.restype = C.c_uint64
        L.oracle_interleave.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32]
        L.oracle_quantise.restype = C.c_uint32
        L.oracle_quantise.argtypes = [C.c_float, C.c_float, C.c_float]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


class Oracle:
    """fp64 Barnes-Hut state (user order).  Inputs are promoted exactly."""

    def __init__(self, mass, pos, vel=None, *, theta, eps, G=1.0, dt=1e-3, k0=0, multipole=1):
        L = lib()
        self.n = int(np.asarray(mass).shape[0])
        self._m = np.ascontiguousarray(mass, dtype=np.float64)
        p = np.ascontiguousarray(np.asarray(pos, dtype=np.float64).reshape(self.n, 3))
        v = None if vel is None else np.ascontiguousarray(np.asarray(vel, dtype=np.float64).reshape(self.n, 3))
        self._h = L.oracle_create(self.n, _p(self._m), _p(p), None if v is None else _p(v),
                                  float(theta), float(eps), float(G), float(dt), int(k0))
        if not self._h:
            raise OracleError(OR_ERR_ARG, "oracle_create failed")
        if multipole != 1:
            self._chk(L.oracle_set_multipole(self._h, int(multipole)))
        self.built = False

    def close(self):
        if self._h:
            lib().oracle_destroy(self._h)
            self._h = None

    __del__ = close

    def _chk(self, rc):
        if rc != OR_OK:
            raise OracleError(rc, lib().oracle_last_error(self._h).decode())

    def build(self):
        self._chk(lib().oracle_build(self._h))
        self.built = True
        return self

    def root(self):
        lo = np.zeros(3, np.float32)
        Lv = np.zeros(1, np.float32)
        sc = np.zeros(1, np.float32)
        self._chk(lib().oracle_root(self._h, _p(lo), _p(Lv), _p(sc)))
        return lo, Lv[0], sc[0]

    def keys(self):
        k = np.zeros(self.n, np.uint64)
        perm = np.zeros(self.n, np.int64)
        self._chk(lib().oracle_get_keys(self._h, _p(k), _p(perm)))
        return k, perm

    def tree(self, with_moments=False):
        n_nodes = lib().oracle_get_tree(self._h, None, None, None, None, None, 0)
        if n_nodes < 0:
            raise OracleError(OR_ERR_ARG, "tree not built")
        lv = np.zeros(n_nodes, np.uint8)
        fi = np.zeros(n_nodes, np.int64)
        co = np.zeros(n_nodes, np.int64)
        M = np.zeros(n_nodes, np.float64) if with_moments else None
        MX = np.zeros((n_nodes, 3), np.float64) if with_moments else None
        lib().oracle_get_tree(self._h, _p(lv), _p(fi), _p(co),
                              _p(M) if with_moments else None, _p(MX) if with_moments else None, n_nodes)
        if with_moments:
            return lv, fi, co, M, MX
        return lv, fi, co

    def quadrupoles(self):
        """Q[node, 6] (xx yy zz xy xz yz) in the tree export order (multipole = 2)."""
        k = lib().oracle_get_quadrupoles(self._h, None, 0)
        if k < 0:
            raise OracleError(OR_ERR_ARG, "no quadrupoles (multipole = 1 or tree not built)")
        Q = np.zeros((k, 6), np.float64)
        lib().oracle_get_quadrupoles(self._h, _p(Q), k)
        return Q

    def forces(self, targets=None):
        """(acc[nt,3] fp64 with G applied, interactions[nt]) for user-index targets."""
        if targets is None:
            nt = self.n
            t = None
        else:
            t = np.ascontiguousarray(targets, dtype=np.int64)
            nt = t.shape[0]
        acc = np.zeros((nt, 3), np.float64)
        cnt = np.zeros(nt, np.int64)
        self._chk(lib().oracle_forces(self._h, nt, None if t is None else _p(t), _p(acc), _p(cnt)))
        return acc, cnt

    def step(self, nsteps=1):
        inter = np.zeros(nsteps, np.int64)
        self._chk(lib().oracle_step(self._h, int(nsteps), _p(inter)))
        return inter

    def step_targets(self, targets):
        """One leapfrog step of the given user-index targets from the current
        state, without advancing it: (pos[nt,3], vel[nt,3], interactions[nt])."""
        t = np.ascontiguousarray(targets, dtype=np.int64)
        nt = t.shape[0]
        po = np.zeros((nt, 3), np.float64)
        vo = np.zeros((nt, 3), np.float64)
        cnt = np.zeros(nt, np.int64)
        self._chk(lib().oracle_step_targets(self._h, nt, _p(t), _p(po), _p(vo), _p(cnt)))
        self.built = True
        return po, vo, cnt

    def state(self):
        p = np.zeros((self.n, 3), np.float64)
        v = np.zeros((self.n, 3), np.float64)
        lib().oracle_get_state(self._h, _p(p), _p(v))
        return p, v


def direct(mass, pos, eps, G=1.0, targets=None):
    """O(N^2) softened direct sum, fp64."""
    m = np.ascontiguousarray(mass, dtype=np.float64)
    p = np.ascontiguousarray(np.asarray(pos, dtype=np.float64).reshape(-1, 3))
    n = m.shape[0]
    if targets is None:
        t, nt = None, n
    else:
        t = np.ascontiguousarray(targets, dtype=np.int64)
        nt = t.shape[0]
    acc = np.zeros((nt, 3), np.float64)
    rc = lib().oracle_direct(n, _p(m), _p(p), float(eps), float(G), nt, None if t is None else _p(t), _p(acc))
    if rc != OR_OK:
        raise OracleError(rc, "direct sum: eps == 0 with coincident particles")
    return acc


def interleave(qx, qy, qz) -> int:
    return int(lib().oracle_interleave(qx, qy, qz))


def quantise(x, lo, scale) -> int:
    return int(lib().oracle_quantise(x, lo, scale))
