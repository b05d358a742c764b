"""Orders beyond the specialised kernels: moments of orders 9..20 and
cumulants of orders 7..16 run on the any-order kernels (csrc/generic.cu, one
thread per stored element), the reference's full range (symten.hpp:87
kMaxOrder = 20; cumulants.hpp:24 partitions up to s = 16).  Bit-exact
against the CPU port, which tests/test_oracle.py pins to the reference at
these orders too."""
import numpy as np
import pytest

from paper_1701_06446_b200 import capi
from test_gpu_parity import assert_series_bitwise

pytestmark = pytest.mark.gpu

SHAPES = [  # (rows, n, d, b)
    (12, 3, 9, 2),    # generic moments and cumulants 7..9
    (10, 4, 10, 3),   # truncated edge block
    (9, 3, 7, 2),     # d = 7: specialised moment kernels, C_7 generic
    (10, 5, 8, 2),    # d = 8: the specialised kernels' last order, C_7 / C_8 generic
    (8, 2, 12, 1),    # b = 1: every index its own block
    (6, 2, 16, 2),    # the largest order with cumulants (one block, 65536 copies of 17 values)
]
IDS = [f"r{a}_n{b}_d{c}_b{d}" for a, b, c, d in SHAPES]


@pytest.mark.parametrize("shape", SHAPES, ids=IDS)
def test_moments_and_update_bitwise(port, shape):
    rows, n, d, b = shape
    rng = np.random.default_rng(900 + rows + 10 * d)
    x = rng.standard_normal((rows, n)) * 0.9 + 0.2
    p = max(1, rows // 3)
    xin = rng.standard_normal((p, n)) * 0.9
    m = capi.moment_series(x, d, b)
    want = port.moment_series(x, d, b)
    assert_series_bitwise(m.tensors(), want, "moment_series")
    capi.moments_update(m, xin, x[:p])
    port.moments_update(want, rows, xin, x[:p], b)
    assert_series_bitwise(m.tensors(), want, "moments_update")
    top = capi.moment_tensor(x, d, b)
    assert np.array_equal(top, port.moment_tensor(x, d, b))


@pytest.mark.parametrize("shape", [s for s in SHAPES if s[2] <= 10], ids=[i for i, s in zip(IDS, SHAPES) if s[2] <= 10])
def test_cumulants_and_report_bitwise(port, shape):
    rows, n, d, b = shape
    rng = np.random.default_rng(77 + rows + d)
    x = rng.standard_normal((rows, n)) * 0.8 - 0.1
    m = capi.moment_series(x, d, b)
    c = capi.moms2cums(m)
    cw = port.moms2cums(port.moment_series(x, d, b), n, b)
    assert_series_bitwise(c.tensors(), cw, "moms2cums")
    got = capi.window_report(c, 3)
    rep = port.report(cw, n, b, 3, rows)
    for key in ("norm_c1", "norm_c2", "max_abs_skewness", "max_abs_kurtosis"):
        assert got[key] == rep[key], key
    assert sorted(got["nu"]) == list(range(3, d + 1))
    for o, v in rep["nu"].items():
        assert got["nu"][o] == v, o


def test_stream_order_nine(port):
    n, d, b, T, p = 3, 9, 2, 18, 6
    rng = np.random.default_rng(909)
    rows = rng.standard_normal((T + 3 * p, n)) * 0.9
    st = capi.Stream(n, d, T, p, b, rows[:T], resync_every=0)
    m = port.moment_series(rows[:T], d, b)
    for k in range(3):
        rep = st.step(rows[T + k * p: T + (k + 1) * p])
        port.moments_update(m, T, rows[T + k * p: T + (k + 1) * p], rows[k * p: (k + 1) * p], b)
    c = port.moms2cums(m, n, b)
    assert_series_bitwise(st.moments(), m, "stream moments")
    assert_series_bitwise(st.cumulants(), c, "stream cumulants")
    want = port.report(c, n, b, 4, T)
    assert rep["window"] == 4 and rep["nu"] == want["nu"]
    st.close()


def test_order_limits():
    x = np.random.default_rng(1).standard_normal((5, 2))
    m = capi.moment_series(x, 17, 1)  # tensors up to order 20 exist ...
    with pytest.raises(capi.CsbInvalidArgument):
        capi.moms2cums(m)  # ... but partitions stop at s = 16 (cumulants.hpp:24)
    with pytest.raises(capi.CsbInvalidArgument):
        capi.moment_series(x, 21, 1)
    assert "generic" in capi.top_kernel(4, 12, 2)
