"""Sampled bitwise parity at sizes the full CPU pipeline cannot reach
(SURVEY §8c sampled-element oracle).  Test infrastructure.

Stored positions are drawn uniformly over every block of an order (so the
symmetric copies inside diagonal blocks are hit as well as canonical
entries); each maps to its sorted (canonical) index, whose exact value the
oracle recomputes with the reference's per-element arithmetic
(oracle/cumstream_oracle.c: oc_sample_stream_moments, oc_sample_cumulants).
Moments come straight from the window rows; cumulants of order s from the
device's own M_s at those positions and its complete C_1..C_{s-1}, which
are themselves checked one order down -- an inductive check of every order.
"""
from __future__ import annotations

from itertools import combinations_with_replacement
from math import comb

import numpy as np


def block_list(order: int, n: int, b: int):
    """Blocks in lex order of non-decreasing j (symten.cpp:105-140): index
    tuples, extents and offsets."""
    g = (n + b - 1) // b
    idx = np.array(list(combinations_with_replacement(range(g), order)), dtype=np.int64).reshape(-1, order)
    ext = np.minimum(b, n - idx * b)
    vol = np.prod(ext, axis=1)
    off = np.concatenate([[0], np.cumsum(vol)])
    return idx, ext, off


def sample_positions(order: int, n: int, b: int, count: int, rng: np.random.Generator):
    """(stored offsets, sorted indices) of `count` stored positions drawn
    uniformly over the stored elements; exhaustive when the order is small."""
    idx, ext, off = block_list(order, n, b)
    stored = int(off[-1])
    if stored <= count:
        pos = np.arange(stored, dtype=np.int64)
    else:
        pos = np.unique(rng.integers(0, stored, count, dtype=np.int64))
    blk = np.searchsorted(off, pos, side="right") - 1
    rem = pos - off[blk]
    o = np.zeros((pos.size, order), dtype=np.int64)
    for k in range(order - 1, -1, -1):
        e = ext[blk, k]
        o[:, k] = rem % e
        rem //= e
    full = idx[blk] * b + o
    return pos.astype(np.uint64), np.sort(full, axis=1).astype(np.int32)


def check_stream_sampled(port, st, rows: np.ndarray, n: int, d: int, b: int, T: int, p: int, steps: int,
                         count: int, seed: int = 0, lower_full_limit: int = 200_000_000) -> dict:
    """Every sampled stored element of M_1..M_d and C_1..C_d of the device
    stream `st` (after prime + `steps` updates of the rows) equals the
    reference's value bit for bit.  Returns per-order sample counts."""
    rng = np.random.default_rng(seed)
    checked = {}
    m_at = {}
    for s in range(1, d + 1):
        pos, sidx = sample_positions(s, n, b, count, rng)
        got = st.gather("M", s, pos)
        want = port.sample_stream_moments(rows, T, p, steps, s, s == d, sidx)
        bad = np.flatnonzero(got != want)
        assert bad.size == 0, (f"M{s}: {bad.size} of {pos.size} sampled elements differ "
                               f"(first: index {sidx[bad[0]].tolist()} got {got[bad[0]]!r} want {want[bad[0]]!r})")
        m_at[s] = (pos, sidx, got)
        checked[f"M{s}"] = int(pos.size)
    c_full = []
    for s in range(1, d + 1):
        pos, sidx, mval = m_at[s]
        got = st.gather("C", s, pos)
        if s == 1:
            want = mval  # C_1 = M_1 (cumulants.cpp:139)
        else:
            want = port.sample_cumulants(c_full, n, b, s, sidx, mval)
        bad = np.flatnonzero(got != want)
        assert bad.size == 0, (f"C{s}: {bad.size} of {pos.size} sampled elements differ "
                               f"(first: index {sidx[bad[0]].tolist()} got {got[bad[0]]!r} want {want[bad[0]]!r})")
        checked[f"C{s}"] = int(pos.size)
        if s < d:
            stored = block_list(s, n, b)[2][-1]
            assert stored <= lower_full_limit, "lower order too large to download"
            c_full.append(st.download("C", s))
    return checked


def canonical_count(n: int, s: int) -> int:
    return comb(n + s - 1, s)
