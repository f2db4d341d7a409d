"""The reference's C++ API driving the GPU library through include/sad_b200_compat.hpp, checked
against the reference in one process (tests/cpp/compat_check.cpp, built by oracle/Makefile where
/root/reference exists; the binary ships with the repo)."""
import os
import subprocess

import pytest

BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "compat_check")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(BIN), reason="compat_check not built (needs /root/reference at build time)")
def test_reference_cpp_api_on_gpu():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
