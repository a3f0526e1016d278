"""Thin ctypes binding of libbh.so (include/bh.h) -- argument marshalling only.

Every step of the Barnes-Hut path runs in the CUDA kernels of csrc/; this module
only allocates the device workspace with torch (PyTorch is plumbing: device
memory, streams, process groups), passes pointers and sizes, and raises on a
non-zero bh_status.  There is no CPU fallback: if libbh.so is missing or no
CUDA device is visible, every entry point raises.

Names follow the ABI: bh_create / bh_set_state / bh_build_tree /
bh_compute_forces / bh_step / bh_sync / bh_destroy and the bh_get_* getters.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BH_LIB") or os.path.join(_HERE, "lib", "libbh.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "bh.h")

BH_OK, BH_ERR_ARG, BH_ERR_CUDA, BH_ERR_OOM, BH_ERR_STATE, BH_ERR_NONFINITE, BH_ERR_NCCL = 0, -1, -2, -3, -4, -5, -6
BH_HOST, BH_DEVICE = 0, 1
PHASES = ("bbox", "keys_sort", "tree", "moments", "walk", "exchange")


class BhParams(C.Structure):
    _fields_ = [
        ("n", C.c_int64),
        ("theta", C.c_double),
        ("eps", C.c_double),
        ("G", C.c_double),
        ("dt", C.c_double),
        ("device", C.c_int),
        ("rank", C.c_int),
        ("world", C.c_int),
        ("stream", C.c_void_p),
        ("nccl_comm", C.c_void_p),
        ("workspace", C.c_void_p),
        ("workspace_bytes", C.c_size_t),
        ("node_capacity", C.c_int64),
        ("walk_group", C.c_int),
        ("multipole", C.c_int),
    ]


class BhStats(C.Structure):
    _fields_ = [
        ("n_records", C.c_int64),
        ("n_internal", C.c_int64),
        ("node_capacity", C.c_int64),
        ("interactions", C.c_int64),
        ("mac_fallbacks", C.c_int64),
        ("own_begin", C.c_int64),
        ("own_end", C.c_int64),
        ("steps", C.c_int64),
        ("opens", C.c_int64),
        ("interactions_cum", C.c_int64),
        ("opens_cum", C.c_int64),
        ("record_visits", C.c_int64),
        ("redo_targets", C.c_int64),
        ("near_sorted", C.c_int64),
        ("sort_bad_keys", C.c_int64),
        ("leaf_visits", C.c_int64),
    ]


class BhError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_names.get(code, code)}: {msg}")
        self.code = code


_names = {0: "BH_OK", -1: "BH_ERR_ARG", -2: "BH_ERR_CUDA", -3: "BH_ERR_OOM", -4: "BH_ERR_STATE",
          -5: "BH_ERR_NONFINITE", -6: "BH_ERR_NCCL"}
_lib = None


def load_library(path: str = LIB_PATH):
    """Load libbh.so; raises if it has not been built (no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise ImportError(f"{path} not built: run `python -m paper_1109_5190_b200.build` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(path)
        vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int
        P = C.POINTER(BhParams)
        sig = {
            "bh_workspace_bytes": (C.c_size_t, [P]),
            "bh_create": (i32, [C.POINTER(vp), P, vp, vp, vp, i32]),
            "bh_set_state": (i32, [vp, vp, vp, vp, i32]),
            "bh_build_tree": (i32, [vp]),
            "bh_compute_forces": (i32, [vp, vp, i32]),
            "bh_step": (i32, [vp, i32]),
            "bh_advance": (i32, [vp, vp, vp, vp, i32, vp, vp, i32]),
            "bh_sync": (i32, [vp]),
            "bh_destroy": (i32, [vp]),
            "bh_get_state": (i32, [vp, vp, vp, i32]),
            "bh_get_root": (i32, [vp, vp, vp, vp]),
            "bh_get_keys": (i32, [vp, vp, vp]),
            "bh_get_tree": (i32, [vp, vp, vp, vp, i64, C.POINTER(i64)]),
            "bh_get_moments": (i32, [vp, vp, vp, i64]),
            "bh_get_interactions": (i32, [vp, vp, vp]),
            "bh_get_own": (i32, [vp, vp, vp, i32]),
            "bh_get_own_cost": (i32, [vp, vp, i32]),
            "bh_get_quadrupoles": (i32, [vp, vp, i64, C.POINTER(i64)]),
            "bh_get_pos4": (i32, [vp, vp, i64, i64, i32]),
            "bh_set_pos4": (i32, [vp, vp, i64, i64, i32]),
            "bh_set_partition": (i32, [vp, vp, vp, i32]),
            "bh_get_pos4_ptr": (i32, [vp, C.POINTER(vp)]),
            "bh_set_peers": (i32, [vp, vp]),
            "bh_step_phase": (i32, [vp, i32]),
            "bh_get_stats": (i32, [vp, C.POINTER(BhStats)]),
            "bh_set_profiling": (i32, [vp, i32]),
            "bh_set_walk_stats": (i32, [vp, i32]),
            "bh_get_profile": (i32, [vp, vp, vp, vp]),
            "bh_last_error": (C.c_char_p, [vp]),
            "bh_status_string": (C.c_char_p, [i32]),
            "bh_nccl_unique_id": (i32, [vp]),
            "bh_nccl_comm_init": (i32, [C.POINTER(vp), vp, i32, i32, i32]),
            "bh_nccl_comm_destroy": (i32, [vp]),
            "bh_nccl_comm_info": (i32, [vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _ptr(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(C.c_void_p)
    return C.c_void_p(a.data_ptr())  # torch tensor


def _host_f32(a, shape):
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a.reshape(shape)


class BarnesHut:
    """One bh_ctx: a Barnes-Hut simulation state on one device (one rank)."""

    def __init__(self, mass, pos, vel=None, *, theta, eps, G=1.0, dt=1e-3, device=0, rank=0, world=1,
                 nccl_comm=None, node_capacity=0, walk_group=0, stream=None, multipole=1):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("BarnesHut needs a CUDA device (B200, sm_100a); there is no CPU fallback")
        self.L = load_library()
        self.torch = torch
        on_dev = isinstance(pos, torch.Tensor) and pos.is_cuda
        n = int(mass.shape[0])
        self.n = n
        self.device = device
        torch.cuda.set_device(device)
        # a dedicated (non-default) stream: all of the ctx's work is enqueued on it and
        # callers time it with events recorded on self.stream
        self.stream = stream if stream is not None else torch.cuda.Stream(device)
        p = BhParams(n=n, theta=float(theta), eps=float(eps), G=float(G), dt=float(dt), device=device, rank=rank,
                     world=world, stream=C.c_void_p(self.stream.cuda_stream), nccl_comm=nccl_comm,
                     workspace=None, workspace_bytes=0, node_capacity=int(node_capacity),
                     walk_group=int(walk_group), multipole=int(multipole))
        nbytes = self.L.bh_workspace_bytes(C.byref(p))
        if nbytes == 0:
            raise BhError(BH_ERR_ARG, "invalid parameters")
        self.workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device=f"cuda:{device}")
        if os.environ.get("BH_POISON_WORKSPACE"):
            # test hook: every byte 0xFF (NaN as fp32 / fp64, huge as an index),
            # so a kernel reading memory nothing wrote this step shows up
            self.workspace.fill_(0xFF)
        base = self.workspace.data_ptr()
        p.workspace = (base + 255) & ~255
        p.workspace_bytes = nbytes
        self.params = p
        h = C.c_void_p()
        # the workspace comes from torch's caching allocator, ordered on the
        # caller's current stream (a reused block may still be in use there, and
        # the poison fill runs there): the ctx stream starts after it
        self.stream.wait_stream(torch.cuda.current_stream(device))
        if on_dev:
            m_, p_, v_ = (mass.contiguous().float(), pos.contiguous().float(),
                          None if vel is None else vel.contiguous().float())
            rc = self.L.bh_create(C.byref(h), C.byref(p), _ptr(m_), _ptr(p_), _ptr(v_), BH_DEVICE)
        else:
            m_, p_ = _host_f32(mass, (n,)), _host_f32(pos, (n, 3))
            v_ = None if vel is None else _host_f32(vel, (n, 3))
            rc = self.L.bh_create(C.byref(h), C.byref(p), _ptr(m_), _ptr(p_), _ptr(v_), BH_HOST)
        if rc != BH_OK:
            raise BhError(rc, self.L.bh_last_error(None).decode())
        self.h = h

    # ------------------------------------------------------------------ utils
    def _chk(self, rc):
        if rc != BH_OK:
            raise BhError(rc, self.L.bh_last_error(self.h).decode())

    def _release_peer_workspaces(self):
        # other ranks' workspaces opened by dist.share_replicas (CUDA IPC): unmapped
        # here, after this ctx's last store into them, never at interpreter exit
        # (a mapping torn down after the CUDA context is gone can crash the exit)
        if getattr(self, "_peer_workspaces", None):
            self.sync()
            self._peer_workspaces = None

    def close(self):
        if getattr(self, "h", None):
            self._release_peer_workspaces()
            self.L.bh_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ ABI
    def set_state(self, mass, pos, vel=None):
        """Replace positions / velocities (user order); `mass` None keeps the
        current masses, `vel` None means zero velocities."""
        torch = self.torch
        if isinstance(pos, torch.Tensor) and pos.is_cuda:
            self._keep = (None if mass is None else mass.contiguous().float(), pos.contiguous().float(),
                          None if vel is None else vel.contiguous().float())
            self.stream.wait_stream(torch.cuda.current_stream(self.device))
            self._chk(self.L.bh_set_state(self.h, *map(_ptr, self._keep), BH_DEVICE))
        else:
            n = self.n
            m_ = None if mass is None else _host_f32(mass, (n,))
            p_ = _host_f32(pos, (n, 3))
            v_ = None if vel is None else _host_f32(vel, (n, 3))
            self._chk(self.L.bh_set_state(self.h, _ptr(m_), _ptr(p_), _ptr(v_), BH_HOST))
            self._chk(self.L.bh_sync(self.h))

    def build_tree(self):
        self._chk(self.L.bh_build_tree(self.h))

    def compute_forces(self, out=None):
        """Accelerations [n,3] (user order).  `out`: a CUDA tensor to fill
        asynchronously; default returns a host numpy array."""
        if out is not None:
            cur = self.torch.cuda.current_stream(self.device)
            self.stream.wait_stream(cur)
            self._chk(self.L.bh_compute_forces(self.h, _ptr(out), BH_DEVICE))
            cur.wait_stream(self.stream)  # the caller's stream sees the result
            return out
        a = np.zeros((self.n, 3), np.float32)
        self._chk(self.L.bh_compute_forces(self.h, _ptr(a), BH_HOST))
        return a

    def step(self, nsteps=1):
        self._chk(self.L.bh_step(self.h, int(nsteps)))

    def advance(self, mass, pos, vel, nsteps=1, pos_out=None, vel_out=None):
        """set_state(mass, pos, vel) + step(nsteps) + get_state in one call
        (bh_advance: the velocity upload overlaps the first tree build).  Host
        arrays in -> host arrays out (allocated if not given); CUDA tensors in ->
        CUDA tensors out (pos_out / vel_out required, or None to skip).
        `mass` None keeps the masses, `vel` None means zero velocities."""
        torch = self.torch
        n = self.n
        if isinstance(pos, torch.Tensor) and pos.is_cuda:
            keep = (None if mass is None else mass.contiguous().float(), pos.contiguous().float(),
                    None if vel is None else vel.contiguous().float())
            cur = torch.cuda.current_stream(self.device)
            self.stream.wait_stream(cur)
            self._chk(self.L.bh_advance(self.h, _ptr(keep[0]), _ptr(keep[1]), _ptr(keep[2]), int(nsteps),
                                        _ptr(pos_out), _ptr(vel_out), BH_DEVICE))
            cur.wait_stream(self.stream)
            return pos_out, vel_out
        m_ = None if mass is None else _host_f32(mass, (n,))
        p_ = _host_f32(pos, (n, 3))
        v_ = None if vel is None else _host_f32(vel, (n, 3))
        if pos_out is None:
            pos_out = np.zeros((n, 3), np.float32)
        if vel_out is None:
            vel_out = np.zeros((n, 3), np.float32)
        self._chk(self.L.bh_advance(self.h, _ptr(m_), _ptr(p_), _ptr(v_), int(nsteps), _ptr(pos_out), _ptr(vel_out),
                                    BH_HOST))
        return pos_out, vel_out

    def sync(self):
        self._chk(self.L.bh_sync(self.h))

    def get_state(self, pos_out=None, vel_out=None):
        if pos_out is not None or vel_out is not None:
            cur = self.torch.cuda.current_stream(self.device)
            self.stream.wait_stream(cur)
            self._chk(self.L.bh_get_state(self.h, _ptr(pos_out), _ptr(vel_out), BH_DEVICE))
            cur.wait_stream(self.stream)
            return pos_out, vel_out
        pos = np.zeros((self.n, 3), np.float32)
        vel = np.zeros((self.n, 3), np.float32)
        self._chk(self.L.bh_get_state(self.h, _ptr(pos), _ptr(vel), BH_HOST))
        return pos, vel

    def get_root(self):
        lo = np.zeros(3, np.float32)
        Lv = np.zeros(1, np.float32)
        sc = np.zeros(1, np.float32)
        self._chk(self.L.bh_get_root(self.h, _ptr(lo), _ptr(Lv), _ptr(sc)))
        return lo, Lv[0], sc[0]

    def get_keys(self):
        k = np.zeros(self.n, np.uint64)
        perm = np.zeros(self.n, np.uint32)
        self._chk(self.L.bh_get_keys(self.h, _ptr(k), _ptr(perm)))
        return k, perm

    def get_tree(self):
        nn = C.c_int64(0)
        rc = self.L.bh_get_tree(self.h, None, None, None, 0, C.byref(nn))
        if rc not in (BH_OK, BH_ERR_ARG):
            self._chk(rc)
        m = nn.value
        lv = np.zeros(m, np.uint8)
        fi = np.zeros(m, np.uint32)
        co = np.zeros(m, np.uint32)
        self._chk(self.L.bh_get_tree(self.h, _ptr(lv), _ptr(fi), _ptr(co), m, C.byref(nn)))
        return lv, fi, co

    def get_moments(self):
        nn = C.c_int64(0)
        rc = self.L.bh_get_tree(self.h, None, None, None, 0, C.byref(nn))
        if rc not in (BH_OK, BH_ERR_ARG):
            self._chk(rc)
        m = nn.value
        M = np.zeros(m, np.float64)
        MX = np.zeros((m, 3), np.float64)
        self._chk(self.L.bh_get_moments(self.h, _ptr(M), _ptr(MX), m))
        return M, MX

    def get_quadrupoles(self):
        """fp64 Q[node, 6] (xx yy zz xy xz yz) in get_tree order (multipole = 2)."""
        nn = C.c_int64(0)
        self._chk(self.L.bh_get_quadrupoles(self.h, None, 0, C.byref(nn)))
        Q = np.zeros((nn.value, 6), np.float64)
        self._chk(self.L.bh_get_quadrupoles(self.h, _ptr(Q), nn.value, C.byref(nn)))
        return Q

    def get_interactions(self):
        c = np.zeros(self.n, np.uint32)
        tot = C.c_uint64(0)
        self._chk(self.L.bh_get_interactions(self.h, _ptr(c), C.c_void_p(C.addressof(tot))))
        return c, int(tot.value)

    def get_own(self):
        """(icount[own], vel[own][3]) of this rank's own slice, storage order."""
        st = self.get_stats()
        m = int(st["own_end"] - st["own_begin"])
        c = np.zeros(m, np.uint32)
        v = np.zeros((m, 3), np.float32)
        self._chk(self.L.bh_get_own(self.h, _ptr(c), _ptr(v), BH_HOST))
        return c, v

    def get_own_cost(self):
        """trips[own]: the last walk's loop trips of each own particle's group
        (bh_get_own_cost; the walk-time cost for dist.rebalance)."""
        st = self.get_stats()
        m = int(st["own_end"] - st["own_begin"])
        t = np.zeros(m, np.uint32)
        self._chk(self.L.bh_get_own_cost(self.h, _ptr(t), BH_HOST))
        return t

    def get_pos4(self, lo, hi):
        """Storage-order slice [lo, hi) of the replicated (x, y, z, m)."""
        out = np.zeros((max(0, hi - lo), 4), np.float32)
        self._chk(self.L.bh_get_pos4(self.h, _ptr(out), int(lo), int(hi), BH_HOST))
        return out

    def set_pos4(self, a, lo, hi):
        a = np.ascontiguousarray(a, dtype=np.float32).reshape(-1, 4)
        self._chk(self.L.bh_set_pos4(self.h, _ptr(a), int(lo), int(hi), BH_HOST))

    def pos4_ptr(self) -> int:
        """Device address of this ctx's pos4 replica (inside self.workspace)."""
        out = C.c_void_p()
        self._chk(self.L.bh_get_pos4_ptr(self.h, C.byref(out)))
        return int(out.value)

    def set_peers(self, pos4_of_rank):
        """The fused exchange (bh_set_peers): every rank's pos4 replica as a device
        address on this ctx's device (this rank's entry ignored); None = off."""
        if pos4_of_rank is None:
            self._chk(self.L.bh_set_peers(self.h, None))
            self._release_peer_workspaces()
            return
        arr = (C.c_void_p * len(pos4_of_rank))(*[int(x) if x else None for x in pos4_of_rank])
        self._chk(self.L.bh_set_peers(self.h, C.cast(arr, C.c_void_p)))

    def step_phase(self, phase):
        """Half a step: 0 = build the tree (K0-K5), 1 = walk + leapfrog + exchange."""
        self._chk(self.L.bh_step_phase(self.h, int(phase)))

    def set_partition(self, bounds, vel_own):
        """New ownership bounds[world + 1] and the new own slice's velocities."""
        b = np.ascontiguousarray(bounds, dtype=np.int64)
        v = np.ascontiguousarray(vel_own, dtype=np.float32).reshape(-1, 3)
        self._chk(self.L.bh_set_partition(self.h, _ptr(b), _ptr(v) if v.size else None, BH_HOST))

    def get_stats(self) -> dict:
        s = BhStats()
        self._chk(self.L.bh_get_stats(self.h, C.byref(s)))
        return {f: getattr(s, f) for f, _ in BhStats._fields_}

    def set_walk_stats(self, on=True):
        self._chk(self.L.bh_set_walk_stats(self.h, 1 if on else 0))

    def set_profiling(self, on=True):
        self._chk(self.L.bh_set_profiling(self.h, 1 if on else 0))

    def get_profile(self) -> dict:
        ms = np.zeros(6, np.float64)
        ln = np.zeros(6, np.int64)
        calls = np.zeros(1, np.int64)
        self._chk(self.L.bh_get_profile(self.h, _ptr(ms), _ptr(ln), _ptr(calls)))
        return {"ms": dict(zip(PHASES, ms.tolist())), "launches": dict(zip(PHASES, ln.tolist())),
                "calls": int(calls[0])}


# module-level aliases with the ABI names
def bh_create(mass, pos, vel=None, **kw) -> BarnesHut:
    return BarnesHut(mass, pos, vel, **kw)


def bh_build_tree(ctx: BarnesHut):
    ctx.build_tree()


def bh_compute_forces(ctx: BarnesHut, out=None):
    return ctx.compute_forces(out)


def bh_step(ctx: BarnesHut, nsteps=1):
    ctx.step(nsteps)


def bh_destroy(ctx: BarnesHut):
    ctx.close()


def nccl_unique_id() -> bytes:
    L = load_library()
    buf = (C.c_ubyte * 128)()
    rc = L.bh_nccl_unique_id(C.cast(buf, C.c_void_p))
    if rc != BH_OK:
        raise BhError(rc, "ncclGetUniqueId failed")
    return bytes(buf)


def nccl_comm_init(uid: bytes, world: int, rank: int, device: int):
    L = load_library()
    buf = (C.c_ubyte * 128).from_buffer_copy(uid)
    comm = C.c_void_p()
    rc = L.bh_nccl_comm_init(C.byref(comm), C.cast(buf, C.c_void_p), world, rank, device)
    if rc != BH_OK:
        raise BhError(rc, "ncclCommInitRank failed")
    return comm


def nccl_comm_info(comm) -> dict:
    """{"count", "rank", "device"} of an NCCL communicator (bh_nccl_comm_info)."""
    L = load_library()
    cnt, rk, dev = C.c_int(0), C.c_int(0), C.c_int(0)
    rc = L.bh_nccl_comm_info(comm, C.byref(cnt), C.byref(rk), C.byref(dev))
    if rc != BH_OK:
        raise BhError(rc, "ncclCommCount / UserRank / CuDevice failed")
    return {"count": cnt.value, "rank": rk.value, "device": dev.value}


def nccl_comm_destroy(comm):
    load_library().bh_nccl_comm_destroy(comm)
