"""Pins the CPU oracle before anything is checked against it.

* The C restatement (oracle/cumstream_oracle.c) against the committed golden
  vectors produced by the reference itself (tests/golden/make_golden.py):
  bitwise for moments and cumulants.
* Against the live reference build (oracle/_ref) on fresh random cases.
* Known-answer tests restated from the reference's own unit tests
  (/root/reference/proj/tests/*.cpp, cited per test).
"""
import glob
import math
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = sorted(glob.glob(os.path.join(HERE, "golden", "*.npz")))


def load(path):
    z = np.load(path)
    return {k: z[k] for k in z.files}


def replay_port(port, g):
    n, d, b, T, p, steps = (int(g[k]) for k in ("n", "d", "b", "T", "p", "steps"))
    stream = g["stream"]
    m = port.moment_series(stream[:T], d, b)
    prime = [x.copy() for x in m]
    reports = []
    for k in range(steps):
        xin = stream[T + k * p: T + (k + 1) * p]
        # ring: outgoing rows are the oldest p rows of the current window
        start = k * p
        xout = stream[start: start + p]
        port.moments_update(m, T, xin, xout, b)
        c = port.moms2cums(m, n, b)
        reports.append(port.report(c, n, b, k + 2, T))
    return prime, m, c, reports


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_port_matches_reference_golden(port, path):
    g = load(path)
    d = int(g["d"])
    prime, m, c, reports = replay_port(port, g)
    for s in range(1, d + 1):
        assert np.array_equal(prime[s - 1], g[f"Mprime{s}"]), f"prime M{s}"
        assert np.array_equal(m[s - 1], g[f"M{s}"]), f"M{s}"
        assert np.array_equal(c[s - 1], g[f"C{s}"]), f"C{s}"
    want = g["reports"][-1]
    got = reports[-1]
    assert got["window"] == int(want[0]) and got["rows"] == int(want[1])
    assert got["norm_c1"] == want[2] and got["norm_c2"] == want[3]
    for o in range(3, d + 1):
        assert got["nu"][o] == want[6 + o - 3]


@pytest.mark.parametrize("shape", [(50, 5, 4, 2), (30, 4, 5, 3), (40, 7, 3, 3), (20, 6, 2, 1),
                                   (25, 3, 4, 3), (100, 10, 6, 3), (60, 24, 4, 3), (33, 4, 1, 1)])
def test_port_matches_live_reference(port, ref, shape):
    rows, n, d, b = shape
    rng = np.random.default_rng(rows * 31 + n)
    x = rng.standard_normal((rows, n)) + 0.3
    mp, mr = port.moment_series(x, d, b), ref.moment_series(x, d, b)
    assert all(np.array_equal(a, c) for a, c in zip(mp, mr))
    xi = rng.standard_normal((7, n))
    port.moments_update(mp, rows, xi, x[:7], b)
    ref.moments_update(mr, rows, xi, x[:7], b)
    assert all(np.array_equal(a, c) for a, c in zip(mp, mr))
    cp, cr = port.moms2cums(mp, n, b), ref.moms2cums(mr, n, b)
    assert all(np.array_equal(a, c) for a, c in zip(cp, cr))
    for s in range(1, d + 1):
        assert np.array_equal(port.moment_tensor(x, s, b), ref.moment_tensor(x, s, b))
        kp, kr = port.knorm(cp[s - 1], s, n, b), ref.knorm(cr[s - 1], s, n, b)
        # bitwise vs the v3 build; the v4 (AVX-512) reference differs in the
        # last bits of its own vectorised fold.
        assert abs(kp - kr) <= 1e-14 * abs(kr)


def test_layout_counts(port):
    # test_symten.cpp:32-48 — block counts 3/5/10; 5 = 2+2+1 truncates the corner
    assert port.layout(2, 2, 1)[1] == 3
    assert port.layout(4, 4, 2)[1] == 5
    assert port.layout(3, 5, 2)[1] == 10
    st, nb = port.layout(2, 5, 2)
    assert nb == 6 and st == 4 + 4 + 2 + 4 + 2 + 1


def test_toy_window(port):
    # test_stream.cpp:110-121 — window {3,4,5,6}: mean 4.5, biased variance 1.25
    x = np.array([[1.0], [2.0], [3.0], [4.0]])
    m = port.moment_series(x, 2, 1)
    port.moments_update(m, 4, np.array([[5.0], [6.0]]), np.array([[1.0], [2.0]]), 1)
    c = port.moms2cums(m, 1, 1)
    assert c[0][0] == pytest.approx(4.5, rel=1e-14)
    assert c[1][0] == pytest.approx(1.25, rel=1e-13)


def test_cli_toy_report(port):
    # test_cli.cpp:114-123 — window {1,2,3,4}: norm_c1 2.5, norm_c2 1.25,
    # nu3 0, nu4 = 2.125 / 1.25^2
    x = np.array([[1.0], [2.0], [3.0], [4.0]])
    c = port.moms2cums(port.moment_series(x, 4, 1), 1, 1)
    rep = port.report(c, 1, 1, 1, 4)
    assert rep["norm_c1"] == pytest.approx(2.5, rel=1e-12)
    assert rep["norm_c2"] == pytest.approx(1.25, rel=1e-12)
    assert abs(rep["nu"][3]) < 1e-10
    assert rep["nu"][4] == pytest.approx(2.125 / (1.25 * 1.25), rel=1e-10)


def test_nu_exact(port):
    # test_gauge.cpp:31-43 — c = (0, 4, -16): nu3 = 16 / 4^1.5 = 2 exactly
    c = [np.array([0.0]), np.array([4.0]), np.array([-16.0])]
    assert port.nu(c, 1, 1, 3) == 2.0


def test_population_gaussian_exact_zero(port):
    # test_cumulants.cpp:57-86 — standard Gaussian raw moments -> C3 = C4 = 0 exactly
    n, b = 3, 2

    def dense_to_block(order, f):
        from itertools import product
        st, _ = port.layout(order, n, b)
        # fill through the block layout: enumerate blocks in lex order
        out = np.zeros(st)
        grid = (n + b - 1) // b
        pos = 0
        for j in sorted(set(tuple(sorted(t)) for t in product(range(grid), repeat=order))):
            ext = [min(b, n - jj * b) for jj in j]
            for o in product(*[range(e) for e in ext]):
                out[pos] = f([jj * b + oo for jj, oo in zip(j, o)])
                pos += 1
        assert pos == st
        return out

    d = lambda i, a, c: 1.0 if i[a] == i[c] else 0.0  # noqa: E731
    m = [dense_to_block(1, lambda i: 0.0),
         dense_to_block(2, lambda i: d(i, 0, 1)),
         dense_to_block(3, lambda i: 0.0),
         dense_to_block(4, lambda i: d(i, 0, 1) * d(i, 2, 3) + d(i, 0, 2) * d(i, 1, 3)
                        + d(i, 0, 3) * d(i, 1, 2))]
    c = port.moms2cums(m, n, b)
    assert np.all(c[0] == 0.0) and np.all(c[2] == 0.0) and np.all(c[3] == 0.0)


def test_constant_and_single_sample(port):
    # test_cumulants.cpp:88-107
    c = port.moms2cums(port.moment_series(np.ones((5, 1)), 4, 1), 1, 1)
    assert c[0][0] == 1.0 and c[1][0] == 0.0 and c[2][0] == 0.0 and c[3][0] == 0.0
    one = np.array([[2.0, -1.0, 0.5]])
    c1 = port.moms2cums(port.moment_series(one, 2, 1), 3, 1)
    assert np.all(c1[1] == 0.0)


def test_partition_counts(port):
    # test_partitions.cpp:14-23 — Stirling numbers of the second kind, RGS order
    stirling = {(4, 2): 7, (4, 3): 6, (5, 2): 15, (6, 3): 90, (6, 2): 31, (6, 4): 65}
    for (s, k), v in stirling.items():
        assert len(port.partitions(s, k)) == v
    assert port.partitions(3, 2) == [[[0, 1], [2]], [[0, 2], [1]], [[0], [1, 2]]]
    assert sum(len(port.partitions(6, k)) for k in range(1, 7)) == 203  # Bell(6)


def test_identical_batches_fixed_point(port):
    # test_moments.cpp:144-152 — identical in/out leaves M bitwise unchanged
    rng = np.random.default_rng(5)
    m = port.moment_series(rng.standard_normal((40, 3)), 3, 2)
    before = [t.copy() for t in m]
    batch = rng.standard_normal((8, 3))
    port.moments_update(m, 40, batch, batch, 2)
    assert all(np.array_equal(a, c) for a, c in zip(m, before))


def test_sampled_element_oracle(port):
    import ctypes as C
    lib = port.lib
    lib.oc_sample_moment.restype = C.c_double
    lib.oc_sample_moment.argtypes = [C.POINTER(C.c_double), C.c_size_t, C.c_size_t,
                                     C.POINTER(C.c_int), C.c_int]
    rng = np.random.default_rng(9)
    x = rng.standard_normal((64, 5))
    idx = (C.c_int * 3)(0, 2, 4)
    v = lib.oc_sample_moment(x.ctypes.data_as(C.POINTER(C.c_double)), 64, 5, idx, 3)
    assert math.isclose(v, float(np.mean(x[:, 0] * x[:, 2] * x[:, 4])), rel_tol=1e-13)


def test_exact_sampled_oracle_matches_full_port(port):
    """The exact sampled-element oracle (used by the full-size GPU parity
    tests at cfg2-cfg4) reproduces the full port bit for bit: moments after
    prime + updates, element offsets, cumulants from the lower orders."""
    from itertools import combinations_with_replacement as cwr
    for (n, d, b, T, p, steps) in ((10, 4, 3, 40, 7, 3), (7, 6, 2, 20, 5, 2)):
        rng = np.random.default_rng(n * d)
        x = rng.standard_normal((T + steps * p, n))
        m = port.moment_series(x[:T], d, b)
        for k in range(steps):
            port.moments_update(m, T, x[T + k * p: T + (k + 1) * p], x[k * p: (k + 1) * p], b)
        c = port.moms2cums(m, n, b)
        for s in range(1, d + 1):
            idx = np.array(list(cwr(range(n), s)), dtype=np.int32)
            off = port.element_offsets(s, n, b, idx).astype(np.int64)
            v = port.sample_stream_moments(x, T, p, steps, s, s == d, idx)
            assert np.array_equal(v, m[s - 1][off]), (n, d, s)
            if s >= 2:
                cv = port.sample_cumulants(c[:s - 1], n, b, s, idx, m[s - 1][off])
                assert np.array_equal(cv, c[s - 1][off]), (n, d, s)


HIGH = [(12, 3, 9, 2), (10, 4, 10, 3), (9, 3, 7, 2), (8, 2, 12, 1)]


@pytest.mark.parametrize("shape", HIGH, ids=[f"r{a}_n{b}_d{c}_b{d}" for a, b, c, d in HIGH])
def test_port_matches_live_reference_high_orders(port, ref, shape):
    """Orders above the specialised kernels' range (the any-order device
    kernels are checked against the port in tests/test_gpu_high_order.py)."""
    rows, n, d, b = shape
    rng = np.random.default_rng(4000 + rows + d)
    x = rng.standard_normal((rows, n)) * 0.9 + 0.2
    p = max(1, rows // 3)
    xin = rng.standard_normal((p, n))
    mp, mr = port.moment_series(x, d, b), ref.moment_series(x, d, b)
    port.moments_update(mp, rows, xin, x[:p], b)
    ref.moments_update(mr, rows, xin, x[:p], b)
    for s in range(d):
        assert np.array_equal(mp[s], mr[s]), f"M{s + 1}"
    if d <= 10:
        cp, cr = port.moms2cums(mp, n, b), ref.moms2cums(mr, n, b)
        for s in range(d):
            assert np.array_equal(cp[s], cr[s]), f"C{s + 1}"
        assert port.report(cp, n, b, 2, rows) == ref.report(cr, n, b, 2, rows)
