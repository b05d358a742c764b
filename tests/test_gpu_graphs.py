"""CUDA-graph replay of the stream step (csb_stream_use_graphs): one graph per
(ring head, batch address, report?) key, captured on the key's second visit.
Steps run from a graph must equal eager steps bit for bit -- moments,
cumulants and every window report -- on the host-buffer path, the pipelined
upload path and the device-buffer path, across ring wrap-around, and a
resync step in between must run eagerly without disturbing the cache."""
import numpy as np
import pytest

from shard_stream_case import case_rows

pytestmark = pytest.mark.gpu

CASES = [  # (n, d, b, T, p, steps, seed)
    (24, 4, 3, 64, 16, 25, 51),   # cfg0 geometry: 4 ring heads
    (20, 6, 4, 60, 20, 19, 52),   # order 6 (persistent moms2cums not taken: n != 48)
    (13, 4, 3, 50, 20, 31, 53),   # odd n (DFMA fallback pair kernel), T % p != 0: 5 heads, wrapped segments
    (48, 6, 4, 96, 48, 13, 54),   # cfg2 geometry: tail kernel + persistent order-6 moms2cums
]


def _run(case, graphs, mode, resync_every=0):
    from paper_1701_06446_b200 import capi

    n, d, b, T, p, steps, seed = case
    rows = case_rows(n, T, p, steps, seed)
    st = capi.Stream(n, d, T, p, b, rows[:T], resync_every=resync_every)
    st.use_graphs(graphs)
    reps = []
    keep = []
    for k in range(steps):
        x = np.ascontiguousarray(rows[T + k * p: T + (k + 1) * p])
        if mode == "host":
            reps.append(st.step(x))
        elif mode == "upload":
            st.upload(x)
            reps.append(st.step_uploaded())
        else:
            import torch
            if not keep:
                keep = [torch.empty((p, n), dtype=torch.float64, device="cuda") for _ in range(2)]
            buf = keep[k % 2]
            buf.copy_(torch.from_numpy(x))
            torch.cuda.synchronize()
            st.step_dev(buf.data_ptr(), p, n, report=False)
            reps.append(st.report())
    out = (st.moments(), st.cumulants(), reps, st.graph_replays())
    st.close()
    return out


@pytest.mark.parametrize("mode", ["host", "upload", "dev"])
@pytest.mark.parametrize("case", CASES, ids=[f"n{c[0]}_d{c[1]}_b{c[2]}" for c in CASES])
def test_graph_steps_equal_eager_steps(case, mode):
    m0, c0, r0, n0 = _run(case, False, mode)
    m1, c1, r1, n1 = _run(case, True, mode)
    assert n0 == 0
    assert n1 >= 2, f"no step ran from a graph ({n1} replays)"
    d = case[1]
    for s in range(d):
        assert np.array_equal(m0[s], m1[s]), f"M{s + 1}"
        assert np.array_equal(c0[s], c1[s]), f"C{s + 1}"
    assert r0 == r1


def test_resync_steps_stay_eager():
    case = (24, 4, 3, 64, 16, 25, 55)
    m0, c0, r0, _ = _run(case, False, "host", resync_every=5)
    m1, c1, r1, n1 = _run(case, True, "host", resync_every=5)
    assert n1 >= 1
    for s in range(4):
        assert np.array_equal(m0[s], m1[s]) and np.array_equal(c0[s], c1[s])
    assert r0 == r1


def test_graphs_survive_scratch_growth():
    """A captured graph holds raw scratch pointers; a larger shape used in
    between reallocates the scratch, so the graph must be dropped and
    captured again (generation check), not replayed on freed memory."""
    from paper_1701_06446_b200 import capi

    case = (24, 4, 3, 64, 16, 30, 56)
    n, d, b, T, p, steps, seed = case
    rows = case_rows(n, T, p, steps, seed)

    def run(graphs, disturb):
        st = capi.Stream(n, d, T, p, b, rows[:T], resync_every=0)
        st.use_graphs(graphs)
        reps = []
        for k in range(steps):
            if disturb and k == 14:  # graphs are replaying by now: grow the scratch under them
                # more tiles than any shape this process has run: the DMMA stash must grow
                big = np.random.default_rng(1).standard_normal((64, 56))
                capi.moments_update(capi.moment_series(big, 6, 4), big[:16], big[16:32])
            reps.append(st.step(rows[T + k * p: T + (k + 1) * p]))
        out = (st.moments(), st.cumulants(), reps, st.graph_replays())
        st.close()
        return out

    m0, c0, r0, _ = run(False, False)
    m1, c1, r1, n1 = run(True, True)
    assert n1 >= 4
    assert r0 == r1
    for s in range(d):
        assert np.array_equal(m0[s], m1[s]) and np.array_equal(c0[s], c1[s])
