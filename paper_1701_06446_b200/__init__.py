"""cumstream_b200: B200-native sliding-window moment/cumulant update
(arXiv 1701.06446) behind the reference's C++ interface.

The product is the in-tree C-ABI library lib/libcumstream_b200.so (CUDA
kernels for sm_100a + host runtime, sources in csrc/), declared in
include/cumstream_b200.h.  `capi` is its Python FFI.
"""
from . import capi  # noqa: F401

__all__ = ["capi"]
