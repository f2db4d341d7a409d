"""The device ports of glibc's exp / expf (sad_device.cuh) against the host libm the reference links:
the fit's double tables, stats softmax and seeding logits and its fp32 softmax go through them, so any
ulp difference would break bit-identity of whole fits."""
import ctypes as C
import math

import numpy as np
import pytest

import paper_2604_21984_b200 as sad

pytestmark = pytest.mark.gpu


def _dev(G, x, which):
    """which: 0 exp, 1 expf, 2 log (the device ports of sad_device.cuh)."""
    y = np.empty_like(x)
    G._call("math_exp", x.ctypes.data_as(C.POINTER(C.c_double)), y.ctypes.data_as(C.POINTER(C.c_double)),
            C.c_size_t(x.size), C.c_int(int(which)))
    return y


def _glibc_exp(x):
    """This host's libm exp (what the reference links), overflow to inf without a Python exception."""
    import ctypes.util
    libm = C.CDLL(ctypes.util.find_library("m"))
    libm.exp.restype = C.c_double
    libm.exp.argtypes = [C.c_double]
    return np.array([libm.exp(float(v)) for v in x])


def test_double_exp_matches_glibc():
    G = sad.gpu_backend(0)
    rng = np.random.default_rng(7)
    parts = [-rng.random(1_000_000) * 60.0,            # softmax weights
             (rng.random(1_000_000) - 0.5) * 44.0,     # tables: exp(log tau), exp(+-a)
             (rng.random(300_000) - 0.5) * 1420.0,     # full range incl. |x| > 512
             (rng.random(100_000) - 0.5) * 1e-6,
             np.array([0.0, -0.0, 1e-300, -1e-300, 709.78, -745.1, 710.0, -746.0, np.inf, -np.inf])]
    x = np.ascontiguousarray(np.concatenate(parts))
    y = _dev(G, x, False)
    ref = _glibc_exp(x)
    # every input, the special-case range |x| > 512 (subnormal and huge results) included
    assert np.array_equal(y.view(np.uint64), ref.view(np.uint64))
    # dense sample of the k < 0 special case (weights of far candidates in the fp64 softmax)
    xs = np.ascontiguousarray(-512.0 - rng.random(2_000_000) * 233.2)
    ys = _dev(G, xs, False)
    rs = _glibc_exp(xs)
    assert np.array_equal(ys.view(np.uint64), rs.view(np.uint64))


def test_double_log_matches_glibc():
    """sad_dlog (densify's split anisotropy, budget.cpp:198-199) against this host's libm log: the
    densify ratio range, the near-1 polynomial path, the whole normal range, subnormals and specials."""
    import ctypes.util
    G = sad.gpu_backend(0)
    rng = np.random.default_rng(9)
    x = np.ascontiguousarray(np.concatenate([
        1.05 * np.exp(rng.random(1_000_000) * np.log(1e18 / 1.05)),
        (1.0 - 2.0 ** -4) + rng.random(1_000_000) * (2.0 ** -4 + float.fromhex("0x1.09p-4")),
        np.exp((rng.random(300_000) - 0.5) * 1400.0),
        rng.random(1000) * 1e-310,
        np.array([1.0, 2.0, 0.5, 1e18, 1.05, 1e300, np.inf, 0.0])]))
    y = _dev(G, x, 2)
    libm = C.CDLL(ctypes.util.find_library("m"))
    libm.log.restype = C.c_double
    libm.log.argtypes = [C.c_double]
    ref = np.array([libm.log(float(v)) for v in x])
    assert np.array_equal(y.view(np.uint64), ref.view(np.uint64))


def test_float_expf_matches_glibc():
    G = sad.gpu_backend(0)
    rng = np.random.default_rng(8)
    xf = np.concatenate([-rng.random(500_000).astype(np.float32) * 100,
                         (rng.random(200_000).astype(np.float32) - 0.5) * 170]).astype(np.float32)
    y = _dev(G, xf.astype(np.float64), True).astype(np.float32)
    ref = np.exp(xf)  # numpy float32 exp goes to... not glibc expf; compare with math via float32 rounding of libm expf
    import ctypes.util
    libm = C.CDLL(ctypes.util.find_library("m"))
    libm.expf.restype = C.c_float
    libm.expf.argtypes = [C.c_float]
    sample = np.arange(0, xf.size, 7)
    ref = np.array([libm.expf(float(v)) for v in xf[sample]], dtype=np.float32)
    assert np.array_equal(y[sample].view(np.uint32), ref.view(np.uint32))
