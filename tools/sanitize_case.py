"""Small streams through every kernel family for compute-sanitizer runs
(racecheck / synccheck / memcheck, one tool per call): the smoke shape
(DMMA top pair, TMA low-order kernel, staged moms2cums), the cfg1 geometry
(<96,6,8>), and the cfg2 geometry (<48,10,4>, the CUDA-core tail kernel,
the persistent order-6 moms2cums)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1701_06446_b200 import capi  # noqa: E402

CASES = [(12, 4, 3, 64, 8, 2), (96, 4, 8, 120, 40, 1), (48, 6, 4, 45, 41, 1)]
for n, d, b, T, p, steps in CASES[: int(sys.argv[1]) if len(sys.argv) > 1 else len(CASES)]:
    rng = np.random.default_rng(n * d)
    rows = rng.standard_normal((T + steps * p, n))
    st = capi.Stream(n, d, T, p, b, rows[:T], resync_every=0)
    for k in range(steps):
        rep = st.step(rows[T + k * p: T + (k + 1) * p])
    print(f"n={n} d={d} b={b}: window {rep['window']} nu{d}={rep['nu'][d]:.6g} kernels={capi.launch_count()}",
          flush=True)
    st.close()
print("sanitize case done")
