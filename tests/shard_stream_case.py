"""One rank of a sharded stream whose exchange runs through the
library's communicator interface backed by torch.distributed gloo
(csb_comm_init_ops, host-staged).  Launched twice by
tests/test_gpu_shards.py (world size 2, both ranks on cuda:0: the ranks'
kernels never wait on each other, the exchange is host-side).  Writes the
rank's owned M_d / C_d ranges, its full lower orders and its reports.

    python tests/shard_stream_case.py RANK WORLD PORT OUT.npz n d b T p steps seed
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (ROOT, HERE):
    if p not in sys.path:
        sys.path.insert(0, p)


def case_rows(n, T, p, steps, seed):
    rng = np.random.default_rng(seed)
    L = rng.uniform(-1.0, 1.0, (n, n))
    chol = np.linalg.cholesky(L @ L.T + 0.5 * np.eye(n))
    return rng.standard_normal((T + steps * p, n)) @ chol.T


def main():
    rank, world, port = (int(v) for v in sys.argv[1:4])
    out = sys.argv[4]
    n, d, b, T, p, steps, seed = (int(v) for v in sys.argv[5:12])
    import torch.distributed as dist

    from paper_1701_06446_b200 import capi

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    capi.check(capi.lib().csb_set_device(0))
    capi.comm_init_torch()
    capi.comm_selftest(1000)  # the library's own check of the exchange interface
    rows = case_rows(n, T, p, steps, seed)
    st = capi.Stream(n, d, T, p, b, rows[:T], resync_every=0, shard_index=rank, shard_count=world)
    capi.comm_destroy()  # the stream keeps its communicator alive (refcount)
    reps = [st.report()]
    for k in range(steps):
        reps.append(st.step(rows[T + k * p: T + (k + 1) * p]))
    m, c = st.moments(), st.cumulants()
    res = {}
    for which, order in ((0, d), (1, d - 1)):
        _, _, lo, hi = capi.shard_range(d, n, b, rank, world, which)
        res[f"range{order}"] = np.array([lo, hi])
    for s in range(1, d + 1):
        res[f"M{s}"] = m[s - 1]
        res[f"C{s}"] = c[s - 1]
    res["nu"] = np.array([[r["nu"][o] for o in range(3, d + 1)] for r in reps])
    res["norms"] = np.array([[r["norm_c1"], r["norm_c2"], r.get("max_abs_skewness", 0.0),
                              r.get("max_abs_kurtosis", 0.0)] for r in reps])
    part = np.empty(capi.layout_size(d, n, b)[1])
    fb = capi._u64()
    capi.check(capi.lib().csb_stream_norm_partials(st.h, d, capi._dptr(part), part.size, capi.C.byref(fb)))
    res["partials"] = part
    res["first_block"] = np.array([fb.value])
    # tensor dumps from sharded state: gather the owners' block ranges
    st.gather_shards()
    res[f"M{d}_gathered"] = st.moments()[d - 1]
    res[f"C{d}_gathered"] = st.cumulants()[d - 1]
    st.close()
    np.savez(out, **res)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
