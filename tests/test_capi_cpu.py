"""CPU-side checks of the C-ABI library: it exists, loads, exports every
symbol include/cumstream_b200.h declares, and fails loudly (no CPU
fallback) when asked to compute without a GPU."""
import ctypes
import os

import numpy as np
import pytest

from paper_1701_06446_b200 import capi
from csb_helpers import gpu_available


def test_library_built_and_loads():
    assert os.path.exists(capi.LIB_PATH), "run __graft_entry__.build()"
    assert capi.lib().csb_version() >= 1


def test_exports_every_header_symbol():
    L = ctypes.CDLL(capi.LIB_PATH)
    syms = capi.header_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing


def test_layout_host_only():
    # SymTensor block counts (test_symten.cpp:32-48), computed without a GPU
    assert capi.layout_size(2, 2, 1)[1] == 3
    assert capi.layout_size(4, 4, 2)[1] == 5
    assert capi.layout_size(3, 5, 2)[1] == 10
    assert capi.layout_size(4, 96, 8) == (5591040, 1365)  # cfg1 M4
    assert capi.layout_size(6, 96, 8) == (3244294144, 12376)  # cfg4 M6


def test_layout_errors_map_to_invalid_argument():
    with pytest.raises(capi.CsbInvalidArgument):
        capi.layout_size(0, 4, 2)
    with pytest.raises(capi.CsbInvalidArgument):
        capi.layout_size(2, 4, 5)


def test_block_multiplicity():
    def mult(j):
        arr = (ctypes.c_int * len(j))(*j)
        out = ctypes.c_uint64()
        capi.check(capi.lib().csb_block_multiplicity(arr, len(j), ctypes.byref(out)))
        return out.value
    assert mult([0, 1, 2, 3]) == 24 and mult([0, 0, 1, 1]) == 6 and mult([2, 2, 2]) == 1
    with pytest.raises(capi.CsbInvalidArgument):
        mult([1, 0])


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU failure path")
def test_no_cpu_fallback():
    assert capi.lib().csb_device_count() == 0
    with pytest.raises(capi.CsbError, match="no CUDA device"):
        capi.moment_series(np.ones((4, 2)), 2, 1)
