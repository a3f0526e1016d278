"""CPU checks of the boundary: libbh.so loads, exports every entry point that
include/bh.h declares, is built for sm_100a, and the product package never
touches the oracle (task rule ③)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bh.h")
PKG = os.path.join(ROOT, "paper_1109_5190_b200")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(bh_[a-z0-9_]+)\s*\(", src)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    from paper_1109_5190_b200 import build

    path = build.build()
    return ctypes.CDLL(path)


def test_header_declares_the_north_star_entry_points():
    names = declared_functions()
    for n in ("bh_create", "bh_build_tree", "bh_compute_forces", "bh_step", "bh_destroy"):
        assert n in names
    assert len(names) >= 20


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_every_symbol():
    from paper_1109_5190_b200 import bh

    L = bh.load_library()
    for n in declared_functions():
        f = getattr(L, n)
        assert f.argtypes is not None, f"binding does not declare {n}"


def test_workspace_size_and_arg_validation(lib):
    from paper_1109_5190_b200.bh import BhParams, load_library

    L = load_library()
    p = BhParams(n=1 << 20, theta=0.5, eps=1e-3, G=1.0, dt=1e-3, device=0, rank=0, world=1)
    b1 = L.bh_workspace_bytes(ctypes.byref(p))
    assert b1 > (1 << 20) * 100
    p.world = 8
    p.rank = 3
    assert 0 < L.bh_workspace_bytes(ctypes.byref(p)) < b1  # velocities for the own slice only
    p.theta = -1
    assert L.bh_workspace_bytes(ctypes.byref(p)) == 0
    p.theta, p.n = 0.5, 0
    assert L.bh_workspace_bytes(ctypes.byref(p)) == 0
    p.n, p.walk_group = 10, 3
    assert L.bh_workspace_bytes(ctypes.byref(p)) == 0
    assert L.bh_status_string(-5) == b"BH_ERR_NONFINITE"


def test_built_for_sm100a(lib):
    from paper_1109_5190_b200 import build

    out = subprocess.run(["cuobjdump", "--list-elf", build.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_product_never_imports_the_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "bh_oracle" not in txt and "liboracle" not in txt, f


def test_no_gpu_means_loud_failure():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1109_5190_b200 import BarnesHut

    with pytest.raises(RuntimeError):
        BarnesHut([1.0], [[0.0, 0.0, 0.0]], theta=0.5, eps=0.1)
