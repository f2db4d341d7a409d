import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA sm_100a) and the built libsad_b200.so")
    config.addinivalue_line("markers", "slow: long-running")


def pytest_sessionfinish(session, exitstatus):
    """With SAD_LIB pointing at the bound-checked build, fail the run if any kernel bound check fired."""
    lib = os.environ.get("SAD_LIB", "")
    if not lib.endswith("_checked.so"):
        return
    try:
        from paper_2604_21984_b200 import api
        if api._gpu is None:
            return
        fails = int(api._gpu.lib.sad_debug_check_failures())
    except Exception:  # noqa: BLE001
        return
    print(f"\nkernel bound-check failures: {fails}")
    if fails != 0:
        session.exitstatus = 1
