"""Bitwise parity of the exact kernels behind the BASELINE configs.

The top-pair launcher picks a specialised DMMA instantiation per shape
(csb_top_kernel): cfg2 (n=48, b=4) runs <48,10,4> with 40-row chunks, cfg3
(n=256, b=16) <256,4,16>, cfg1/cfg4 (n=96, b=8) <96,6,8>.  Two kinds of
check:

* geometry cases -- the config's (n, d, b) and data distribution at a
  reduced window, every pass spanning >= 3 chunks plus a 1..7-row tail
  (the zero-row source of a pass's last chunk), compared element for
  element with the CPU port (M and C in full, or sampled where the full
  port would take minutes);
* full-size cases -- the config's own T and p, prime + 2 steps, checked on
  tens of thousands of sampled stored elements per order with the exact
  sampled-element oracle (tests/sampled.py).
"""
from dataclasses import replace

import numpy as np
import pytest

from sampled import check_stream_sampled

from paper_1701_06446_b200 import capi
from paper_1701_06446_b200.synth import CONFIGS, StreamGen, stream_rows

pytestmark = pytest.mark.gpu


def _rows(cfg, T, p, steps):
    c = replace(CONFIGS[cfg], T=T, p=p)
    return stream_rows(c, steps)


def _stream(rows, n, d, b, T, p, steps):
    st = capi.Stream(n, d, T, p, b, rows[:T], resync_every=0)
    for k in range(steps):
        st.step(rows[T + k * p: T + (k + 1) * p], report=False)
    return st


@pytest.mark.parametrize("T,p", [(125, 41), (167, 127)], ids=["T125_p41", "T167_p127"])
def test_cfg2_kernel_full_compare(port, T, p):
    """<48,10,4>: prime passes of 125 / 167 rows (3 / 4 chunks + 5 / 7),
    update passes of 41 / 127 rows (1 / 3 chunks + 1 / 7); every stored
    element of M_1..M_6 and C_1..C_6."""
    n, d, b = 48, 6, 4
    assert capi.top_kernel(n, d, b) == "moment_top_dmma_kernel<48,10,4>"
    steps = 1
    rows = _rows(2, T, p, steps)
    st = _stream(rows, n, d, b, T, p, steps)
    want = port.moment_series(rows[:T], d, b)
    for k in range(steps):
        port.moments_update(want, T, rows[T + k * p: T + (k + 1) * p], rows[k * p: (k + 1) * p], b)
    got = st.moments()
    for s in range(d):
        bad = np.flatnonzero(got[s] != want[s])
        assert bad.size == 0, f"M{s + 1}: {bad.size} of {got[s].size} differ (first at {bad[0]})"
    cw = port.moms2cums(want, n, b)
    gc = st.cumulants()
    for s in range(d):
        bad = np.flatnonzero(gc[s] != cw[s])
        assert bad.size == 0, f"C{s + 1}: {bad.size} of {gc[s].size} differ (first at {bad[0]})"


def test_cfg2_kernel_series_api_tail(port):
    """csb_moment_series at n=48, b=4 over 45 rows (one chunk + a 5-row tail)."""
    n, d, b = 48, 6, 4
    x = _rows(2, 45, 5, 0)[:45]
    got = capi.moment_series(x, d, b).tensors()
    want = port.moment_series(x, d, b)
    for s in range(d):
        assert np.array_equal(got[s], want[s]), f"M{s + 1}"


def test_cfg3_kernel_sampled(port):
    """<256,4,16>: 16-row chunks; prime 53 rows (3 chunks + 5), updates of
    23 rows (1 chunk + 7), two steps; 2.0e5 sampled elements per order."""
    n, d, b, T, p, steps = 256, 4, 16, 53, 23, 2
    assert capi.top_kernel(n, d, b) == "moment_top_dmma_kernel<256,4,16>"
    rows = _rows(3, T, p, steps)
    st = _stream(rows, n, d, b, T, p, steps)
    got = check_stream_sampled(port, st, rows, n, d, b, T, p, steps, count=200_000, seed=3)
    assert got["M4"] > 150_000 and got["M1"] == 256


def test_cfg1_kernel_geometry_full_compare(port):
    """<96,6,8> (24-row chunks): prime 77 rows (3 chunks + 5), updates of 31
    rows (1 chunk + 7), 2 steps, all stored elements."""
    n, d, b, T, p, steps = 96, 4, 8, 77, 31, 2
    assert capi.top_kernel(n, d, b) == "moment_top_dmma_kernel<96,6,8>"
    rows = _rows(1, T, p, steps)
    st = _stream(rows, n, d, b, T, p, steps)
    want = port.moment_series(rows[:T], d, b)
    for k in range(steps):
        port.moments_update(want, T, rows[T + k * p: T + (k + 1) * p], rows[k * p: (k + 1) * p], b)
    got = st.moments()
    for s in range(d):
        assert np.array_equal(got[s], want[s]), f"M{s + 1}"
    cw = port.moms2cums(want, n, b)
    gc = st.cumulants()
    for s in range(d):
        assert np.array_equal(gc[s], cw[s]), f"C{s + 1}"


FULL = [  # (config, steps, samples per order)
    (1, 2, 100_000),
    (2, 2, 40_000),
    (3, 2, 20_000),
    (4, 2, 8_000),
]


@pytest.mark.parametrize("cfg,steps,count", FULL, ids=[CONFIGS[c].name for c, _, _ in FULL])
def test_full_size_sampled(port, cfg, steps, count):
    """The config's own window and update length, prime + 2 steps, sampled
    stored elements of every order bitwise (cfg4: M_6 is 25.95 GB, about
    55 GB of device state with C)."""
    c = CONFIGS[cfg]
    gen = StreamGen(c)
    rows = np.concatenate([gen.window()] + [gen.batch(k) for k in range(1, steps + 1)])
    st = _stream(rows, c.n, c.d, c.b, c.T, c.p, steps)
    rep = st.report()
    assert all(np.isfinite(v) for v in rep["nu"].values())
    got = check_stream_sampled(port, st, rows, c.n, c.d, c.b, c.T, c.p, steps, count=count, seed=cfg)
    assert got[f"M{c.d}"] > count // 2
    st.close()


@pytest.mark.parametrize("shape", [(16, 6, 8), (16, 5, 8), (24, 5, 8)], ids=["n16_d6_b8", "n16_d5_b8", "n24_d5_b8"])
def test_cfg4_moms2cums_path_full_compare(port, shape):
    """cfg4's cumulant conversion (b = 8, orders 5 and 6): the sub-blocks of a
    block (210 KB / 2.1 MB) cannot be staged, so full blocks run the
    list-driven global-load path moms2cums_v2<S, false, 8>.  Whole-array
    bitwise compare of M and C at a small n with the same block geometry
    (the full-size sampled check is test_full_size_sampled[cfg4])."""
    n, d, b = shape
    T, p = 40, 13
    rng = np.random.default_rng(8600 + n + d)
    rows = rng.standard_normal((T + p, n)) * 0.9 + 0.15
    m = capi.moment_series(rows[:T], d, b)
    capi.moments_update(m, rows[T:], rows[:p])
    want = port.moment_series(rows[:T], d, b)
    port.moments_update(want, T, rows[T:], rows[:p], b)
    c = capi.moms2cums(m)
    cw = port.moms2cums(want, n, b)
    for s in range(d):
        assert np.array_equal(m.tensors()[s], want[s]), f"M{s + 1}"
        assert np.array_equal(c.tensors()[s], cw[s]), f"C{s + 1}"
