"""Soak run for the lock-free kernels: the same window update (and cumulant
conversion) from the same state, hundreds of times, must give one digest.
    python tools/soak.py   (round 2: 150/300/600/40 runs at four shapes, one digest each;
    profiles/r02/soak.txt)"""
import sys, hashlib, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from paper_1701_06446_b200 import capi
def digest(series):
    h = hashlib.sha256()
    for t in series.tensors(): h.update(t.tobytes())
    return h.hexdigest()
for (n, d, b, T, p, reps) in [(48, 6, 4, 240, 87, 150), (96, 4, 8, 400, 130, 300), (24, 4, 3, 300, 50, 600), (48, 6, 4, 2000, 500, 40)]:
    rng = np.random.default_rng(n * 100 + d)
    x = rng.standard_normal((T, n)) * 1.1 + 0.1
    xin = rng.standard_normal((p, n))
    base = capi.moment_series(x, d, b)
    work = capi.Series(n, d, b)
    sm, sc = set(), set()
    for _ in range(reps):
        work.copy_from(base); work.window_len = T
        capi.moments_update(work, xin, x[:p])
        sm.add(digest(work)); sc.add(digest(capi.moms2cums(work)))
    print((n, d, b, T, p), "runs", reps, "distinct M digests", len(sm), "distinct C digests", len(sc), flush=True)
    assert len(sm) == 1 and len(sc) == 1
print("soak ok")
