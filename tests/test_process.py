"""The `cumstream process` path end to end: rows in a
CSV file -> CsvBatchSource -> run() -> one report_json_line per window, via
the C++ drop-in API (paper_1701_06446_b200/cpp/tests/process_main.cpp).
Two runs must be byte-identical and equal to prime()/step() fed the same
batches directly (the reference's acceptance check 8 shape)."""
import os
import subprocess

import pytest

from csb_helpers import gpu_available

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_1701_06446_b200", "lib", "process_b200")

pytestmark = pytest.mark.skipif(not os.path.exists(BIN), reason="process check not built")


@pytest.mark.skipif(gpu_available(), reason="CPU-only expectation")
def test_process_fails_loudly_without_gpu():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=120)
    assert r.returncode == 2 and "no CUDA device" in r.stderr


@pytest.mark.gpu
def test_process_jsonl_deterministic_and_exact():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 6 and all('"nu":{"3":' in ln for ln in lines)
