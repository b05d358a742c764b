"""Parity of the CUDA path (through the C ABI) with the CPU oracle.

The oracle (oracle/cumstream_oracle.c) is pinned bit for bit to the
reference (tests/test_oracle.py), so every `bitwise` assertion below is a
bit-exact match with the reference library on the same inputs.  Norms are
reduced in a different (deterministic, parallel) order than the reference's
sequential fold, so they are held to a relative 1e-13.  The north-star bar
is 1e-10 relative.
"""
import glob
import os

import numpy as np
import pytest

from csb_helpers import rel_gap
from paper_1701_06446_b200 import capi

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = sorted(glob.glob(os.path.join(HERE, "golden", "*.npz")))

SHAPES = [  # (rows, n, d, b): shapes of test_moments.cpp:52-53 and friends
    (50, 5, 4, 2), (30, 4, 5, 3), (40, 7, 3, 3), (20, 6, 2, 1), (25, 3, 4, 3),
    (100, 10, 6, 3), (60, 24, 4, 3), (33, 4, 1, 1), (64, 17, 4, 8), (80, 9, 6, 4),
    (45, 12, 5, 5), (70, 20, 3, 7), (16, 40, 3, 16), (3, 8, 4, 8),
]


def assert_series_bitwise(got, want, what):
    for s, (g, w) in enumerate(zip(got, want), start=1):
        assert g.shape == w.shape, f"{what} order {s} shape"
        if not np.array_equal(g, w):
            bad = np.flatnonzero(g != w)
            raise AssertionError(f"{what} order {s}: {bad.size} of {g.size} differ, "
                                 f"rel_gap={rel_gap(g, w):.3e}, first at {bad[0]}: "
                                 f"{g[bad[0]]!r} vs {w[bad[0]]!r}")


@pytest.mark.parametrize("shape", SHAPES, ids=[f"r{a}_n{b}_d{c}_b{d}" for a, b, c, d in SHAPES])
def test_moment_series_bitwise(port, shape):
    rows, n, d, b = shape
    rng = np.random.default_rng(rows * 7 + n * 3 + d)
    x = rng.standard_normal((rows, n)) + 0.25
    got = capi.moment_series(x, d, b)
    assert got.window_len == rows
    assert_series_bitwise(got.tensors(), port.moment_series(x, d, b), "moment_series")


@pytest.mark.parametrize("shape", SHAPES[:8], ids=[f"r{a}_n{b}_d{c}_b{d}" for a, b, c, d in SHAPES[:8]])
def test_moment_tensor_bitwise(port, shape):
    rows, n, d, b = shape
    rng = np.random.default_rng(rows + n)
    x = rng.standard_normal((rows, n))
    for s in range(1, d + 1):
        got = capi.moment_tensor(x, s, b)
        want = port.moment_tensor(x, s, b)
        assert np.array_equal(got, want), f"order {s}: rel_gap {rel_gap(got, want):.3e}"


@pytest.mark.parametrize("shape", SHAPES, ids=[f"r{a}_n{b}_d{c}_b{d}" for a, b, c, d in SHAPES])
def test_update_and_moms2cums_bitwise(port, shape):
    rows, n, d, b = shape
    rng = np.random.default_rng(rows * 13 + n)
    x = rng.standard_normal((rows, n)) * 1.5 - 0.1
    p = max(1, rows // 5)
    xin = rng.standard_normal((p, n))
    m = capi.moment_series(x, d, b)
    capi.moments_update(m, xin, x[:p])
    want = port.moment_series(x, d, b)
    port.moments_update(want, rows, xin, x[:p], b)
    assert_series_bitwise(m.tensors(), want, "moments_update")
    c = capi.moms2cums(m)
    cw = port.moms2cums(want, n, b)
    assert_series_bitwise(c.tensors(), cw, "moms2cums")
    for s in range(1, d + 1):
        for k in (1.0, 2.0, 3.0):
            kg, kw = capi.knorm(c, s, k), port.knorm(cw[s - 1], s, n, b, k)
            assert abs(kg - kw) <= 1e-13 * abs(kw) + 1e-300, (s, k, kg, kw)
    if d >= 3:
        for o in range(3, d + 1):
            try:
                want_nu = port.nu(cw, n, b, o)
            except Exception:
                continue
            assert abs(capi.nu(c, o) - want_nu) <= 1e-13 * abs(want_nu)
    if d >= 2:
        got = capi.window_report(c, 7)
        rep = port.report(cw, n, b, 7, rows)
        assert got["window"] == 7
        for key in ("norm_c1", "norm_c2", "max_abs_skewness", "max_abs_kurtosis"):
            if key in rep:
                assert abs(got[key] - rep[key]) <= 1e-13 * abs(rep[key]), key
        for o, v in rep["nu"].items():
            assert abs(got["nu"][o] - v) <= 1e-13 * abs(v)


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_stream_matches_reference_golden(path):
    """prime + steps through the device stream engine vs the reference's own
    stream run (fixtures written by tests/golden/make_golden.py)."""
    g = np.load(path)
    n, d, b, T, p, steps = (int(g[k]) for k in ("n", "d", "b", "T", "p", "steps"))
    stream = g["stream"]
    st = capi.Stream(n, d, T, p, b, stream[:T])
    for k in range(steps):
        rep = st.step(stream[T + k * p: T + (k + 1) * p])
    assert st.window == steps + 1
    assert_series_bitwise(st.moments(), [g[f"M{s}"] for s in range(1, d + 1)], "stream M")
    assert_series_bitwise(st.cumulants(), [g[f"C{s}"] for s in range(1, d + 1)], "stream C")
    want = g["reports"][-1]
    assert rep["window"] == int(want[0]) and rep["rows"] == int(want[1])
    assert abs(rep["norm_c1"] - want[2]) <= 1e-13 * abs(want[2])
    assert abs(rep["norm_c2"] - want[3]) <= 1e-13 * abs(want[3])
    for o in range(3, d + 1):
        assert abs(rep["nu"][o] - want[6 + o - 3]) <= 1e-12 * abs(want[6 + o - 3]) + 1e-300
    np.testing.assert_array_equal(st.materialize(), stream[steps * p: steps * p + T])


def test_identical_batches_fixed_point():
    # test_moments.cpp:144-152
    rng = np.random.default_rng(5)
    m = capi.moment_series(rng.standard_normal((40, 3)), 3, 2)
    before = m.tensors()
    batch = rng.standard_normal((8, 3))
    capi.moments_update(m, batch, batch)
    assert_series_bitwise(m.tensors(), before, "fixed point")


def test_refeeding_outgoing_rows_is_fixed_point():
    # test_stream.cpp:123-137
    rng = np.random.default_rng(2)
    first = rng.standard_normal((30, 3))
    st = capi.Stream(3, 4, 30, 5, 2, first)
    before = st.moments()
    st.step(first[:5])
    assert_series_bitwise(st.moments(), before, "re-feed")


def test_toy_step():
    # test_stream.cpp:110-121: window {3,4,5,6} -> mean 4.5, variance 1.25
    st = capi.Stream(1, 2, 4, 2, 1, np.array([[1.0], [2.0], [3.0], [4.0]]))
    rep = st.step(np.array([[5.0], [6.0]]))
    c = st.cumulants()
    assert st.window == 2
    assert abs(c[0][0] - 4.5) <= 1e-14 * 4.5 and abs(c[1][0] - 1.25) <= 1e-13 * 1.25
    assert abs(rep["norm_c1"] - 4.5) <= 1e-12


def test_rows_read_metering():
    # test_moments.cpp:182-196, test_stream.cpp:230-243
    rng = np.random.default_rng(3)
    x = rng.standard_normal((25, 3))
    base = capi.rows_read()
    capi.moment_tensor(x, 3, 1)
    assert capi.rows_read() - base == 25
    m = capi.moment_series(x, 3, 1)
    assert capi.rows_read() - base == 50
    up = rng.standard_normal((5, 3))
    capi.moments_update(m, up, up)
    assert capi.rows_read() - base == 60
    st = capi.Stream(3, 3, 25, 5, 1, x)
    b0 = capi.rows_read()
    st.step(up, report=False)
    assert capi.rows_read() - b0 == 10


def test_resync_is_bitwise_recompute(port):
    # test_stream.cpp:171-200: a resync step equals moment_series(materialize())
    rng = np.random.default_rng(8)
    n, d, b, T, p = 5, 4, 2, 40, 8
    rows = rng.standard_normal((T + 3 * p, n))
    st = capi.Stream(n, d, T, p, b, rows[:T], resync_every=3)
    for k in range(3):
        st.step(rows[T + k * p: T + (k + 1) * p], report=False)
    window = st.materialize()
    assert_series_bitwise(st.moments(), port.moment_series(window, d, b), "resync")


def test_errors_map_to_reference_exceptions():
    rng = np.random.default_rng(1)
    x = rng.standard_normal((10, 3))
    m = capi.moment_series(x, 3, 1)
    with pytest.raises(capi.CsbInvalidArgument):
        capi.moments_update(m, rng.standard_normal((11, 3)), rng.standard_normal((11, 3)))
    with pytest.raises(capi.CsbInvalidArgument):
        capi.moments_update(m, rng.standard_normal((2, 4)), rng.standard_normal((2, 4)))
    with pytest.raises(capi.CsbInvalidArgument):
        capi.moment_series(np.zeros((0, 3)), 3, 1)
    c = capi.moms2cums(capi.moment_series(np.ones((4, 1)), 3, 1))
    with pytest.raises(capi.CsbDomainError):
        capi.nu(c, 3)
    with pytest.raises(capi.CsbInvalidArgument):
        capi.nu(c, 2)
    with pytest.raises(capi.CsbInvalidArgument):
        capi.Stream(3, 4, 10, 11, 1, x)


def test_cfg0_full_size(port):
    """BASELINE config 0 at full size: prime + 3 steps, bitwise vs the oracle."""
    from paper_1701_06446_b200.synth import CONFIGS, StreamGen
    cfg = CONFIGS[0]
    g = StreamGen(cfg)
    first = g.window()
    st = capi.Stream(cfg.n, cfg.d, cfg.T, cfg.p, cfg.b, first)
    want = port.moment_series(first, cfg.d, cfg.b)
    ring = first.copy()
    for k in range(1, 4):
        xin = g.batch(k)
        rep = st.step(xin)
        port.moments_update(want, cfg.T, xin, ring[:cfg.p], cfg.b)
        ring = np.concatenate([ring[cfg.p:], xin])
    assert_series_bitwise(st.moments(), want, "cfg0 M")
    cw = port.moms2cums(want, cfg.n, cfg.b)
    assert_series_bitwise(st.cumulants(), cw, "cfg0 C")
    r = port.report(cw, cfg.n, cfg.b, 4, cfg.T)
    for o in (3, 4):
        assert abs(rep["nu"][o] - r["nu"][o]) <= 1e-12 * abs(r["nu"][o])


def test_pipelined_upload_matches_step():
    """csb_stream_upload / csb_stream_step_uploaded (batch k+1's copy
    in flight during step k) give the same states and reports as step()."""
    from paper_1701_06446_b200 import capi
    rng = np.random.default_rng(77)
    n, d, b, T, p, steps = 24, 4, 3, 96, 24, 5
    rows = rng.standard_normal((T + steps * p, n))
    a = capi.Stream(n, d, T, p, b, rows[:T], resync_every=0)
    c = capi.Stream(n, d, T, p, b, rows[:T], resync_every=0)
    batches = [rows[T + k * p: T + (k + 1) * p].copy() for k in range(steps)]
    c.upload(batches[0])
    for k in range(steps):
        ra = a.step(batches[k])
        if k + 1 < steps:
            c.upload(batches[k + 1])
        rc = c.step_uploaded()
        assert ra == rc
    for x, y in zip(a.moments(), c.moments()):
        assert np.array_equal(x, y)
    with pytest.raises(capi.CsbInvalidArgument):
        c.step_uploaded()  # nothing uploaded
