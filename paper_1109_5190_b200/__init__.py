"""B200-native Barnes-Hut force step (arxiv 1109.5190 hot path).

The product is libbh.so (csrc/, C ABI in include/bh.h); `bh` is its thin
ctypes binding.  PyTorch is used only for device memory, streams and process
groups.  There is no CPU fallback.
"""
from .bh import (BH_DEVICE, BH_HOST, BarnesHut, BhError, bh_build_tree, bh_compute_forces, bh_create,  # noqa: F401
                 bh_destroy, bh_step, load_library)

__all__ = ["BarnesHut", "BhError", "bh_create", "bh_build_tree", "bh_compute_forces", "bh_step", "bh_destroy",
           "load_library", "BH_HOST", "BH_DEVICE"]
