"""The bound-checked build of the library (libsad_b200_checked.so: the same sources with -DSAD_CHECKED=1;
shared-memory table indices of the tile reductions, record-pool and overflow-pool indices, owner-merge
records and every site id read from a candidate list are tested inside the kernels and violations counted
on the device).  compute-sanitizer is closed on the GPU pool this runs on, so this is its stand-in: every
kernel (tools/sanitize_driver.py) and the parity suites that force the reduction fallbacks run on the checked
build, and must end with zero bound-check failures and results equal to the reference."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2604_21984_b200", "libsad_b200_checked.so")


def _env():
    if not os.path.exists(CHECKED):
        pytest.skip("checked build missing (__graft_entry__.build builds it)")
    env = dict(os.environ)
    env["SAD_LIB"] = CHECKED
    return env


def test_every_kernel_on_checked_build():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_driver.py")], env=_env(), cwd=ROOT,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "kernel bound-check failures: 0" in r.stdout


def test_parity_suites_on_checked_build():
    suites = ["tests/test_gpu_parity.py", "tests/test_reduction_paths.py", "tests/test_strips.py",
              "tests/test_tau_diffusion.py"]
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider", *suites],
                       env=_env(), cwd=ROOT, capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "kernel bound-check failures: 0" in r.stdout


_FIRE = r"""
import numpy as np, paper_2604_21984_b200 as sad
from tests.fixtures import random_model
G = sad.gpu_backend(0)
big = random_model(40, 32, 100, 1)
f = sad.CandidateField(); f.resize(40, 32, 8)
G.refresh(big, f, sad.RefreshMode.Full, 2, 4, 1, sad.RunOpts(fp64=False))   # capacity >= 100 sites
small = random_model(40, 32, 50, 2)
f2 = sad.CandidateField(); f2.resize(40, 32, 8)
G.refresh(small, f2, sad.RefreshMode.Full, 2, 4, 1, sad.RunOpts(fp64=False))
assert G.lib.sad_debug_check_failures() == 0
ids = f2.ids.reshape(-1, 8).copy(); ids[17, 0] = 60                          # a site id past the store (< capacity)
f2.ids = ids.reshape(-1).copy()
G.propagate_pass(small, f2, sad.PassSpec(1, sad.Stencil.Axial), 4, 9, sad.RunOpts(fp64=False))
print("fired", G.lib.sad_debug_check_failures())
"""


def test_checks_fire_on_a_bad_id():
    """The checks are live: a candidate list holding an id past the site store is counted."""
    r = subprocess.run([sys.executable, "-c", _FIRE], env=_env(), cwd=ROOT, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    n = int(r.stdout.split("fired")[-1])
    assert n > 0
