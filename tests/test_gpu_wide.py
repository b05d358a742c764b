"""Bitwise parity at BASELINE-like widths, where the DMMA kernel's wide
tiles (R = 1 and 2 row sets per CTA, up to 16 column tiles, balanced over
the SM sub-partitions) and the pattern-list mirror of full blocks are
exercised; the small shapes of test_gpu_parity.py only reach R = 4/2 tiles.
Rows are Gaussian with BASELINE's covariance construction, fewer of them so
the CPU oracle finishes in seconds.
"""
import pytest

from wide_case import run_case

pytestmark = pytest.mark.gpu

CASES = [  # (n, d, b, T, p, steps, seed)
    (96, 4, 8, 300, 60, 2, 11),    # cfg1 geometry: windows of 12..1 column tiles
    (130, 3, 16, 200, 50, 2, 12),  # > 16 column tiles: split column ranges, edge blocks
    (40, 6, 4, 24, 8, 2, 13),      # cfg2 geometry (order 6, R = 2 and 4 windows)
    (72, 5, 8, 40, 10, 1, 14),     # order 5, full and edge blocks
    (48, 4, 16, 40, 10, 1, 16),    # cfg3 block size: 64K-entry blocks, 1024-thread moms2cums pass
]


@pytest.mark.parametrize("case", CASES, ids=[f"n{c[0]}_d{c[1]}_b{c[2]}" for c in CASES])
def test_wide_stream_bitwise(case):
    run_case(*case)
