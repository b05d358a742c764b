"""The sharded stream engine end to end: two ranks, each a
`csb_stream` primed with shard_index = rank, shard_count = 2, exchanging
through the library's communicator interface (csb_comm_init_ops) backed by
torch.distributed gloo.  The same collectives run over NCCL in production
(csb_comm_init); this exercises the engine's exchange choreography -- which
ranges are gathered (M_{d-1}), which partials and diagonals are reduced --
without a second GPU.  Every owned order-d element, every gathered /
replicated lower order, and every window report must equal the unsharded
stream's bit for bit (reference ownership split: moments.cpp:76-101)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from shard_stream_case import case_rows

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))

CASES = [  # (n, d, b, T, p, steps, seed)
    (24, 4, 3, 64, 16, 3, 31),    # cfg0 geometry, DMMA top pair, diagonal of C_4 sharded
    (20, 6, 4, 40, 8, 2, 32),     # order 6: C_4 diagonal replicated, C_6 sharded
    (96, 4, 8, 120, 40, 2, 33),   # cfg1 geometry
]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("case", CASES, ids=[f"n{c[0]}_d{c[1]}_b{c[2]}" for c in CASES])
def test_sharded_stream_equals_unsharded(case, tmp_path):
    from paper_1701_06446_b200 import capi

    n, d, b, T, p, steps, seed = case
    world, port = 2, _free_port()
    outs = [str(tmp_path / f"rank{r}.npz") for r in range(world)]
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "shard_stream_case.py"), str(r), str(world),
                               str(port), outs[r], *map(str, case)], stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT, text=True) for r in range(world)]
    logs = []
    for pr in procs:
        out, _ = pr.communicate(timeout=600)
        logs.append(out)
    assert all(pr.returncode == 0 for pr in procs), "\n".join(x[-3000:] for x in logs)

    rows = case_rows(n, T, p, steps, seed)
    st = capi.Stream(n, d, T, p, b, rows[:T], resync_every=0)
    reps = [st.report()]
    for k in range(steps):
        reps.append(st.step(rows[T + k * p: T + (k + 1) * p]))
    want_m, want_c = st.moments(), st.cumulants()
    want_nu = np.array([[r["nu"][o] for o in range(3, d + 1)] for r in reps])
    want_norms = np.array([[r["norm_c1"], r["norm_c2"], r.get("max_abs_skewness", 0.0),
                            r.get("max_abs_kurtosis", 0.0)] for r in reps])

    covered = np.zeros(want_m[d - 1].size, dtype=bool)
    for r in range(world):
        got = np.load(outs[r])
        lo, hi = got[f"range{d}"]
        covered[lo:hi] = True
        assert np.array_equal(got[f"M{d}"][lo:hi], want_m[d - 1][lo:hi]), f"rank {r}: owned M{d}"
        assert np.array_equal(got[f"C{d}"][lo:hi], want_c[d - 1][lo:hi]), f"rank {r}: owned C{d}"
        for s in range(1, d):  # M_{d-1} gathered, lower orders replicated; C_1..C_{d-1} complete
            assert np.array_equal(got[f"M{s}"], want_m[s - 1]), f"rank {r}: M{s}"
            assert np.array_equal(got[f"C{s}"], want_c[s - 1]), f"rank {r}: C{s}"
        assert np.array_equal(got["nu"], want_nu), f"rank {r}: nu"
        assert np.array_equal(got["norms"], want_norms), f"rank {r}: norms / diagonals"
        assert int(got["first_block"][0]) == 0
        # csb_stream_gather_shards: the whole M_d / C_d in block order on every rank
        assert np.array_equal(got[f"M{d}_gathered"], want_m[d - 1]), f"rank {r}: gathered M{d}"
        assert np.array_equal(got[f"C{d}_gathered"], want_c[d - 1]), f"rank {r}: gathered C{d}"
        assert np.all(np.isfinite(got["partials"]))
    assert covered.all(), "the shards do not cover M_d"


def test_nccl_communicator_single_rank_selftest():
    """The production transport: libnccl.so.2 resolved at run time, a real
    (one-rank) communicator, and the engine's two collectives -- grouped
    broadcasts of per-rank ranges and a sum allreduce -- on device buffers,
    verified by csb_comm_selftest.  More ranks need more GPUs than this pool
    grants; bench.py --gpus N runs the same self-test on every rank first."""
    from paper_1701_06446_b200 import capi

    capi.check(capi.lib().csb_set_device(0))
    uid = capi.comm_unique_id()
    assert len(uid) == 128
    capi.comm_init(1, 0, uid)
    try:
        capi.comm_selftest(1)
        capi.comm_selftest(100_000)
    finally:
        capi.comm_destroy()
    with pytest.raises(capi.CsbError):
        capi.comm_selftest(16)  # no communicator any more
