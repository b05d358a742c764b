"""Generate the committed golden vectors from the REFERENCE itself.

Runs the unmodified reference library (oracle/_ref, compiled in place from
/root/reference/proj/src by `make -C oracle ref`) through its own stream API
(cumstream::prime / step, /root/reference/proj/include/cumstream/stream.hpp:69,73)
on small seeded inputs and stores inputs + outputs as .npz fixtures.  The
fixtures travel to the GPU box; /root/reference does not.

    python tests/golden/make_golden.py        # rewrites tests/golden/*.npz

The x86-64-v3 build is used so the norms are the v3 bits (see
oracle/cumstream_oracle.c knorm note).
"""
from __future__ import annotations

import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Oracle, RefStream  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

# (name, n, d, b, T, p, steps, seed, distribution)
CASES = [
    ("toy_n1_d2", 1, 2, 1, 4, 2, 1, 0, "toy"),
    ("n5_d4_b2", 5, 4, 2, 40, 8, 4, 11, "normal"),
    ("n4_d5_b3", 4, 5, 3, 30, 5, 3, 12, "normal"),
    ("n7_d3_b3", 7, 3, 3, 24, 6, 3, 13, "normal"),
    ("n6_d6_b2", 6, 6, 2, 20, 4, 2, 14, "normal"),
    ("n3_d4_b3", 3, 4, 3, 12, 3, 3, 15, "normal"),
    ("n12_d4_b3", 12, 4, 3, 200, 25, 3, 16, "gauss_sigma"),
    ("n9_d4_b4", 9, 4, 4, 50, 50, 2, 17, "heavy"),       # full-window turnover
    ("n8_d6_b3", 8, 6, 3, 40, 7, 2, 18, "contaminated"),
    ("n10_d3_b1", 10, 3, 1, 30, 3, 3, 19, "normal"),
]


def rows_for(dist: str, rng: np.random.Generator, rows: int, n: int) -> np.ndarray:
    if dist == "toy":
        return None
    if dist == "normal":
        return rng.standard_normal((rows, n))
    if dist == "gauss_sigma":
        L = rng.uniform(-1, 1, (n, n))
        S = L @ L.T + 0.5 * np.eye(n)
        return rng.standard_normal((rows, n)) @ np.linalg.cholesky(S).T + 0.25
    if dist == "heavy":
        z = rng.standard_normal((rows, n))
        w = rng.chisquare(5, (rows, 1))
        return z / np.sqrt(w / 5.0)
    if dist == "contaminated":
        x = rng.standard_normal((rows, n))
        m = rng.random((rows, n)) < 0.1
        x[m] = rng.laplace(0.0, 1.0, m.sum())
        return x
    raise ValueError(dist)


def main() -> None:
    ref = Oracle("ref", workers=4)
    v3 = os.path.join(ROOT, "oracle", "_ref", "libcumstream_ref_v3.so")
    ref.lib = ctypes.CDLL(v3)
    ref.path = v3
    ref._bind()
    for name, n, d, b, T, p, steps, seed, dist in CASES:
        rng = np.random.default_rng(seed)
        if dist == "toy":
            stream = np.array([[1.0], [2.0], [3.0], [4.0], [5.0], [6.0]])
        else:
            stream = rows_for(dist, rng, T + p * steps, n)
        first = stream[:T]
        st = RefStream(ref, n, d, T, p, b, first)
        reports = [st.step(stream[T + k * p: T + (k + 1) * p]).copy() for k in range(steps)]
        # prime-only moments as a separate fixture column
        m_prime = ref.moment_series(first, d, b)
        out = {"n": n, "d": d, "b": b, "T": T, "p": p, "steps": steps, "stream": stream,
               "reports": np.array(reports)}
        for s in range(1, d + 1):
            out[f"Mprime{s}"] = m_prime[s - 1]
            out[f"M{s}"] = st.moments(s)
            out[f"C{s}"] = st.cumulants(s)
        st.close()
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print("wrote", name)


if __name__ == "__main__":
    main()
