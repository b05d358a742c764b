"""Window reports bit-identical to the reference.

knorm folds each block's entries in storage order and the blocks in block
order (symten.cpp:257-276); the device reproduces that sequence exactly
(knorm_exact_kernel + the sequential fold, the k = 2 fold vectorised like
the reference built for this host: 8-wide with AVX-512, else 4-wide), so
norms, nu and the diagonal statistics equal the reference's bit for bit and
the `process` JSONL (CSV -> CsvBatchSource -> run -> report_json_line) is
byte-identical to the reference's own process path run on the same file
(oracle/ref_process.cpp, the unmodified reference sources; acceptance
check 8's shape, tests/acceptance.cpp:398-451)."""
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OURS = os.path.join(ROOT, "paper_1701_06446_b200", "lib", "process_b200")


def _ref_binary():
    from oracle.oracle import _cpu_has_avx512
    for v in (["v4", "v3"] if _cpu_has_avx512() else ["v3"]):
        p = os.path.join(ROOT, "oracle", "_ref", f"ref_process_{v}")
        if os.path.exists(p):
            return p
    pytest.skip("oracle/_ref/ref_process_* not built (make -C oracle ref)")


CASES = [  # (n, d, b, T, p, windows, seed): cfg0 at full size, order 6, odd n / edge blocks, order 3
    (24, 4, 3, 5000, 500, 6, 41),
    (20, 6, 4, 600, 150, 4, 42),
    (13, 4, 3, 300, 75, 5, 43),
    (30, 5, 7, 400, 100, 4, 44),
    (16, 3, 5, 200, 50, 5, 45),
]


@pytest.mark.parametrize("case", CASES, ids=[f"n{c[0]}_d{c[1]}_b{c[2]}" for c in CASES])
def test_process_jsonl_byte_identical_to_reference(case, tmp_path):
    n, d, b, T, p, windows, seed = case
    rng = np.random.default_rng(seed)
    L = rng.uniform(-1.0, 1.0, (n, n))
    rows = rng.standard_normal((T + (windows - 1) * p, n)) @ np.linalg.cholesky(L @ L.T + 0.5 * np.eye(n)).T
    csv = tmp_path / "rows.csv"
    # shortest round-trip decimals: both parsers read back the same doubles
    with open(csv, "w") as fh:
        for r in rows:
            fh.write(",".join(repr(float(v)) for v in r) + "\n")
    args = [str(csv), str(n), str(d), str(T), str(p), str(b)]
    want = subprocess.run([_ref_binary(), *args], capture_output=True, text=True, timeout=900)
    assert want.returncode == 0, want.stderr[-2000:]
    got = subprocess.run([OURS, *args], capture_output=True, text=True, timeout=600)
    assert got.returncode == 0, got.stderr[-2000:]
    wl, gl = want.stdout.splitlines(), got.stdout.splitlines()
    assert len(wl) == windows and len(gl) == windows
    for k, (a, c) in enumerate(zip(wl, gl)):
        assert a == c, f"window {k + 1}:\n  reference {a}\n  b200      {c}"


DUMP_CASES = [(12, 4, 3, 200, 50, 3, 46), (10, 6, 4, 120, 30, 2, 47), (13, 5, 4, 90, 30, 3, 48)]


@pytest.mark.parametrize("case", DUMP_CASES, ids=[f"n{c[0]}_d{c[1]}_b{c[2]}" for c in DUMP_CASES])
def test_cumulant_dumps_byte_identical_to_reference(case, tmp_path):
    """--dump-cumulants (tools/cumstream.cpp:90-96): every window's to_json(C, w, 1)
    file equals the reference's byte for byte (the sharded
    gather behind the same call is covered by tests/test_gpu_shards.py)."""
    n, d, b, T, p, windows, seed = case
    rng = np.random.default_rng(seed)
    rows = rng.standard_normal((T + (windows - 1) * p, n)) * 1.25 + 0.1
    csv = tmp_path / "rows.csv"
    with open(csv, "w") as fh:
        for r in rows:
            fh.write(",".join(repr(float(v)) for v in r) + "\n")
    dirs = {}
    for name, binary in (("ref", _ref_binary()), ("b200", OURS)):
        dirs[name] = tmp_path / name
        dirs[name].mkdir()
        res = subprocess.run([binary, str(csv), str(n), str(d), str(T), str(p), str(b), str(dirs[name])],
                             capture_output=True, text=True, timeout=600)
        assert res.returncode == 0, res.stderr[-2000:]
        dirs[name + "_out"] = res.stdout
    assert dirs["ref_out"] == dirs["b200_out"]
    for w in range(1, windows + 1):
        a = (dirs["ref"] / f"window_{w}.json").read_bytes()
        c = (dirs["b200"] / f"window_{w}.json").read_bytes()
        assert len(a) > 100 and a == c, f"window {w}: dump differs from the reference's"
