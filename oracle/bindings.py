"""TEST INFRASTRUCTURE ONLY.  ctypes bindings of the two CPU oracles:

* `ref_backend()`  — the unmodified reference library compiled from /root/reference/proj/src
                     (oracle/_ref/libsadref.so, built by oracle/Makefile).  Present wherever it
                     was built here; it travels to the GPU box as a prebuilt file.
* `c_backend()`    — the plain-C restatement (oracle/_ref/libsado.so).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import this module.
"""
from __future__ import annotations

import ctypes as C
import os

from paper_2604_21984_b200.api import Backend

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libsadref.so")
C_SO = os.path.join(HERE, "_ref", "libsado.so")

_cache = {}


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def ref_backend(threads: int = 1) -> Backend:
    key = ("ref", threads)
    if key not in _cache:
        lib = _cache.get("ref_lib") or C.CDLL(REF_SO)
        _cache["ref_lib"] = lib
        lib.sadref_last_error.restype = C.c_char_p
        lib.sadref_fit_info.argtypes = [C.c_void_p] + [C.c_void_p] * 5
        lib.sadref_fit_free.argtypes = [C.c_void_p]
        lib.sadref_seeded_state.restype = C.c_uint32
        lib.sadref_seeded_state.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32]
        lib.sadref_float_to_half.restype = C.c_uint16
        lib.sadref_float_to_half.argtypes = [C.c_float]
        lib.sadref_half_to_float.restype = C.c_float
        lib.sadref_half_to_float.argtypes = [C.c_uint16]
        lib.sadref_psnr_from_loss.restype = C.c_double
        lib.sadref_psnr_from_loss.argtypes = [C.c_double]
        lib.sadref_mse.restype = C.c_double
        _cache[key] = Backend(lib, "sadref_", "ref", threads=threads)
    return _cache[key]


def c_backend() -> Backend:
    if "c" not in _cache:
        lib = C.CDLL(C_SO)
        lib.sado_last_error.restype = C.c_char_p
        lib.sado_seeded_state.restype = C.c_uint32
        lib.sado_seeded_state.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32]
        lib.sado_float_to_half.restype = C.c_uint16
        lib.sado_float_to_half.argtypes = [C.c_float]
        lib.sado_half_to_float.restype = C.c_float
        lib.sado_half_to_float.argtypes = [C.c_uint16]
        lib.sado_psnr_from_loss.restype = C.c_double
        lib.sado_psnr_from_loss.argtypes = [C.c_double]
        _cache["c"] = Backend(lib, "sado_", "c")
    return _cache["c"]


def build(verbose: bool = False) -> None:
    """Compile libsado.so always and libsadref.so when /root/reference is present."""
    import subprocess
    subprocess.run(["make", "-s", "-f", os.path.join(HERE, "Makefile")], check=True,
                   stdout=None if verbose else subprocess.DEVNULL)
