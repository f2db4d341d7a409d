"""The reference's own test suite on the GPU library ("the reference tests re-link against it
unchanged").  tests/reftests/Makefile compiles /root/reference/proj/tests/test_*.cpp as they are (with the
minimal doctest harness tests/reftests/doctest.h) and links them with tests/reftests/sad_link_shim.cpp,
which defines the hot-path functions of namespace `sad` with the reference's exact signatures over the C
ABI of libsad_b200.so — so every refresh / render / backward / Adam / stats / prune / densify / init /
fit the reference's tests make runs on the B200.  The binaries are built here (where /root/reference
exists) into oracle/_ref/reftests/ and shipped with the snapshot.

Expected failures: exactly one case, "golden file bytes are stable" (test_codec.cpp:348), whose fixture
proj/tests/data/golden.sad is absent from the reference checkout.
"""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "reftests")
SUITES = ["test_core", "test_score", "test_candidates", "test_render", "test_grad", "test_quality", "test_train",
          "test_budget", "test_codec"]
EXPECTED_FAIL = {"test_codec": {"golden file bytes are stable"}}


@pytest.mark.parametrize("name", SUITES)
def test_reference_suite_on_gpu_library(name):
    exe = os.path.join(BIN, name)
    if not os.path.exists(exe):
        pytest.skip("reference test binaries not built (make -f tests/reftests/Makefile needs /root/reference)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=1200, cwd=BIN)
    summary = re.search(r"\[reftest\] .*: (\d+) test cases, (\d+) failed, (\d+) checks, (\d+) failed", r.stdout)
    assert summary, r.stdout[-2000:] + r.stderr[-2000:]
    failed = set(re.findall(r"^\[case failed\] (.*)$", r.stderr, re.M))
    print(summary.group(0))
    assert failed == EXPECTED_FAIL.get(name, set()), r.stderr[-4000:]
    assert int(summary.group(1)) > 0 and int(summary.group(3)) > 0
