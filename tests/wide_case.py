"""One stream case at a BASELINE-like width, checked bitwise against the CPU
oracle (test infrastructure; run in-process by tests/test_gpu_wide.py and
as a subprocess when a kernel-selection environment switch is under test).

    python tests/wide_case.py n d b T p steps seed
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (ROOT, HERE):
    if p not in sys.path:
        sys.path.insert(0, p)


def run_case(n, d, b, T, p, steps, seed):
    from oracle.oracle import Oracle
    from paper_1701_06446_b200 import capi

    port = Oracle("port")
    rng = np.random.default_rng(seed)
    L = rng.uniform(-1.0, 1.0, (n, n))
    chol = np.linalg.cholesky(L @ L.T + 0.5 * np.eye(n))
    rows = rng.standard_normal((T + steps * p, n)) @ chol.T
    first = rows[:T]
    st = capi.Stream(n, d, T, p, b, first, resync_every=0)
    want = port.moment_series(first, d, b)
    ring = first.copy()
    rep = None
    for k in range(steps):
        xin = rows[T + k * p: T + (k + 1) * p]
        rep = st.step(xin)
        port.moments_update(want, T, xin, ring[:p], b)
        ring = np.concatenate([ring[p:], xin])
    got = st.moments()
    for s in range(d):
        if not np.array_equal(got[s], want[s]):
            bad = np.flatnonzero(got[s] != want[s])
            raise AssertionError(f"M{s + 1}: {bad.size} of {got[s].size} differ (first at {bad[0]})")
    cw = port.moms2cums(want, n, b)
    gc = st.cumulants()
    for s in range(d):
        if not np.array_equal(gc[s], cw[s]):
            bad = np.flatnonzero(gc[s] != cw[s])
            raise AssertionError(f"C{s + 1}: {bad.size} of {gc[s].size} differ (first at {bad[0]})")
    r = port.report(cw, n, b, d, T)
    for o in range(3, d + 1):
        assert abs(rep["nu"][o] - r["nu"][o]) <= 1e-12 * abs(r["nu"][o]), (o, rep["nu"][o], r["nu"][o])


if __name__ == "__main__":
    a = [int(v) for v in sys.argv[1:8]]
    run_case(*a)
    print("ok")
