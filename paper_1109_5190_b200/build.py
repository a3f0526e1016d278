"""Build libbh.so in-tree with nvcc for sm_100a (no GPU needed to compile).

    python -m paper_1109_5190_b200.build [--force] [--verbose]

Each csrc/*.cu is compiled to an object with
    -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo
(no -use_fast_math: the keys and the fp64 moments rely on IEEE round-to-
nearest intrinsics), then linked into paper_1109_5190_b200/lib/libbh.so against
the NCCL that torch ships (site-packages/nvidia/nccl), so the library and
torch.distributed share one libnccl.so.2 in the process.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libbh.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import nvidia.nccl  # torch's NCCL wheel

    base = os.path.dirname(nvidia.nccl.__file__) if getattr(nvidia.nccl, "__file__", None) else list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def _newer(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None, objdir_name: str = "build") -> str:
    os.makedirs(LIBDIR, exist_ok=True)
    objdir = os.path.join(HERE, objdir_name)
    lib_out = out or LIB
    os.makedirs(objdir, exist_ok=True)
    inc, lib = nccl_dirs()
    headers = glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "bh.h")]
    objs = []
    nvcc = os.environ.get("NVCC", "nvcc")
    for src in sorted(glob.glob(os.path.join(CSRC, "*.cu"))):
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        if force or _newer(obj, [src] + headers + [__file__]):
            cmd = [nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
                   "-Xptxas", "-v" if verbose else "-O3", "-I", inc, "-I", os.path.join(ROOT, "include"),
                   *[f"-D{d}" for d in defines], "-c", src, "-o", obj]
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True)
    if force or _newer(lib_out, objs):
        cmd = [nvcc, *ARCH, "-shared", "-o", lib_out + ".tmp", *objs, "-L", lib, "-l:libnccl.so.2",
               "-Xlinker", f"-rpath,{lib}", "-lcudart"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        os.replace(lib_out + ".tmp", lib_out)
    return lib_out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
