"""Drop-in check: the reference's own doctest unit suites (test_symten,
test_moments, test_cumulants, test_gauge, test_stream, test_partitions,
test_serialize from
/root/reference/proj/tests, compiled in place -- never copied -- by
`make -C paper_1701_06446_b200/cpp refsuite`) built against the
cumstream_b200 C++ headers and linked to the B200 library."""
import os
import re
import subprocess

import pytest

from csb_helpers import gpu_available

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_1701_06446_b200", "lib", "refsuite_b200")

pytestmark = pytest.mark.skipif(not os.path.exists(BIN), reason="refsuite not built (needs /root/reference)")


def run_suite():
    res = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", res.stdout)
    assert m, res.stdout[-2000:] + res.stderr[-2000:]
    return res, int(m.group(1)), int(m.group(2)), int(m.group(3))


@pytest.mark.skipif(gpu_available(), reason="CPU-only expectations")
def test_refsuite_host_cases_pass_without_gpu():
    res, total, passed, failed = run_suite()
    assert total == 59
    # the host-side utilities (layout, ranker, partitions, predictors, ring
    # buffer) pass; everything touching tensors needs the device
    assert passed >= 15
    assert "no CUDA device" in res.stderr


@pytest.mark.gpu
def test_reference_unit_suites_pass_on_b200():
    res, total, passed, failed = run_suite()
    assert total == 59
    assert failed == 0, res.stderr[-4000:]
