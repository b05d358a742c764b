"""Multi-GPU sharding: the block-prefix partitioner (host
logic, CPU), the exchange algebra the library performs with NCCL (checked
with torch.distributed gloo, world size 2, on CPU), and shard-count
independence of the device results (GPU: k shards run one after another on
one device, assembled, must equal the unsharded result bit for bit)."""
import os

import numpy as np
import pytest

from paper_1701_06446_b200 import capi

SHAPES = [(4, 96, 8), (6, 48, 4), (6, 96, 8), (4, 256, 16), (4, 24, 3), (5, 30, 5)]


@pytest.mark.parametrize("shape", SHAPES, ids=[f"d{d}_n{n}_b{b}" for d, n, b in SHAPES])
def test_partition_covers_blocks_contiguously(shape):
    d, n, b = shape
    for count in (1, 2, 3, 4, 8):
        for which, order in ((0, d), (1, d - 1)):
            stored, nblocks = capi.layout_size(order, n, b)
            prev_b, prev_e = 0, 0
            for s in range(count):
                blo, bhi, elo, ehi = capi.shard_range(d, n, b, s, count, which)
                assert blo == prev_b and elo == prev_e and bhi >= blo and ehi >= elo
                prev_b, prev_e = bhi, ehi
            assert prev_b == nblocks and prev_e == stored


def _canonical_weights(d, n, b):
    from itertools import combinations_with_replacement
    from math import comb
    g = (n + b - 1) // b
    w = []
    for j in combinations_with_replacement(range(g), d):
        c, a = 1, 0
        while a < d:
            e = a + 1
            while e < d and j[e] == j[a]:
                e += 1
            c *= comb(min(b, n - j[a] * b) + e - a - 1, e - a)
            a = e
        w.append(c)
    return w


@pytest.mark.parametrize("shape", [(4, 256, 16), (6, 96, 8), (6, 48, 4)])
def test_partition_is_balanced(shape):
    # canonical elements (the DMMA work) per shard within 10% of ideal for
    # the sharded BASELINE configs (cfg3, cfg4, cfg2)
    d, n, b = shape
    w = _canonical_weights(d, n, b)
    tot = sum(w)
    for count in (2, 4, 8):
        share = [sum(w[slice(*capi.shard_range(d, n, b, s, count, 0)[:2])]) / (tot / count)
                 for s in range(count)]
        assert max(share) <= 1.10, share


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d, n, b = 6, 48, 4
    _, nblocks = capi.layout_size(d, n, b)
    rng = np.random.default_rng(7)
    full = rng.standard_normal(nblocks) ** 2          # per-block partial sums of squares
    mine = np.zeros(nblocks)
    blo, bhi, _, _ = capi.shard_range(d, n, b, rank, world, 0)
    mine[blo:bhi] = full[blo:bhi]
    t = torch.from_numpy(mine)
    dist.all_reduce(t)                                  # collective C3 (library: ncclAllReduce)
    ok_sum = np.array_equal(t.numpy(), full)            # x + 0 == x: exact
    # collective C2: order d-1 ranges gathered by per-owner broadcasts
    stored1, _ = capi.layout_size(d - 1, n, b)
    m_full = rng.standard_normal(stored1)
    buf = np.where(np.arange(stored1) >= 0, np.nan, 0.0)
    _, _, elo, ehi = capi.shard_range(d, n, b, rank, world, 1)
    buf[elo:ehi] = m_full[elo:ehi]
    tb = torch.from_numpy(buf)
    for r in range(world):
        _, _, lo, hi = capi.shard_range(d, n, b, r, world, 1)
        seg = tb[lo:hi].clone()
        dist.broadcast(seg, src=r)
        tb[lo:hi] = seg
    ok_gather = np.array_equal(tb.numpy(), m_full)
    q.put((rank, ok_sum, ok_gather))
    dist.destroy_process_group()


def test_exchange_algebra_gloo_world2():
    import multiprocessing as mp
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok1 and ok2 for _, ok1, ok2 in res), res


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(4, 40, 8), (6, 20, 4), (4, 96, 8), (5, 26, 4)])
def test_shard_count_independence(shape):
    d, n, b = shape
    rng = np.random.default_rng(n * d)
    T, p = 64, 16
    x = rng.standard_normal((T, n)) + 0.2
    xin = rng.standard_normal((p, n))
    full = capi.moment_series(x, d, b)
    capi.moments_update(full, xin, x[:p])
    want_m = full.tensors()
    want_c = capi.moms2cums(full).tensors()
    for count in (2, 3, 4):
        got_m = [np.full_like(t, np.nan) for t in want_m]
        got_c = [np.full_like(t, np.nan) for t in want_c]
        for s in range(count):
            m = capi.moment_series(x, d, b)
            capi.moments_update_shard(m, xin, x[:p], s, count)
            part = m.tensors()
            for which, order in ((0, d), (1, d - 1)):
                _, _, lo, hi = capi.shard_range(d, n, b, s, count, which)
                got_m[order - 1][lo:hi] = part[order - 1][lo:hi]
            for order in range(1, d - 1):  # replicated orders
                assert np.array_equal(part[order - 1], want_m[order - 1])
                got_m[order - 1] = part[order - 1]
        for order in range(d):
            assert np.array_equal(got_m[order], want_m[order]), (count, order + 1)
        # moms2cums on the assembled (complete) moments
        mm = capi.Series(n, d, b)
        for order in range(1, d + 1):
            mm.upload(order, got_m[order - 1])
        mm.window_len = full.window_len
        for s in range(count):
            cpart = capi.moms2cums_shard(mm, s, count).tensors()
            _, _, lo, hi = capi.shard_range(d, n, b, s, count, 0)
            got_c[d - 1][lo:hi] = cpart[d - 1][lo:hi]
            for order in range(1, d):
                got_c[order - 1] = cpart[order - 1]
        for order in range(d):
            assert np.array_equal(got_c[order], want_c[order]), (count, order + 1)
