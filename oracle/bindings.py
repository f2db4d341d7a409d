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

from typing import Optional

from paper_2604_21984_b200 import CandidateField, RefreshMode, RunOpts, SiteStore
from paper_2604_21984_b200.api import Backend, _P, _abi, _ptr, _ref
from paper_2604_21984_b200.types import FitResult, HistoryRow, ImageBuffer, TrainConfig

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libsadref.so")
C_SO = os.path.join(HERE, "_ref", "libsado.so")

_cache = {}


class OracleBackend(Backend):
    """The product binding's methods over a CPU oracle library.  kind 'ref' (sadref_: no context,
    trailing worker count, handle-based fit) or 'c' (sado_: no context, one-call fit)."""

    def __init__(self, lib, prefix: str, kind: str, threads: int = 1):
        super().__init__(lib, prefix, ctx=None)
        self.kind = kind
        self.threads = threads

    def _pre(self, name):
        return ()

    def _thr(self):
        return (C.c_int(self.threads),) if self.kind == "ref" else ()

    def decode_render(self, data: bytes, k: int = 8, passes: int = 16, inject: int = 4, seed: int = 1,
                      fp64: bool = False):
        w, h, st = self.decode_sites(data)
        f = CandidateField()
        f.resize(w, h, k)
        self.refresh(st, f, RefreshMode.Full, passes, inject, seed, RunOpts(fp64=fp64))
        return self.render_image(st, f, RunOpts(fp64=fp64)), st

    def _fit(self, target: ImageBuffer, cfg: TrainConfig, init: Optional[SiteStore]) -> FitResult:
        c = cfg.to_c()
        w, h = target.width, target.height
        if self.kind == "ref":
            hd = _P()
            sv = None
            if init is not None:
                sv, keep = init._view()
            self._call("fit", _ptr(target.data), C.c_int(w), C.c_int(h), C.byref(c), _ref(sv), C.byref(hd))
            try:
                n, nh, sc, sec = C.c_size_t(), C.c_int(), C.c_double(), C.c_double()
                ph = (C.c_double * 8)()
                self.lib.sadref_fit_info(hd, C.byref(n), C.byref(nh), C.byref(sc), C.byref(sec), ph)
                res = self._fit_collect(w, h, cfg, int(n.value), int(nh.value), float(sc.value),
                                        lambda sv, fv, hist: self._call("fit_download", hd, sv, fv, hist))
                res.timing = {"total_ms": sec.value * 1e3, "propagate_ms": ph[0], "fwd_bwd_ms": ph[1],
                              "adam_ms": ph[2], "events_ms": ph[3], "refresh_full_ms": ph[4], "init_ms": ph[5]}
                return res
            finally:
                self.lib.sadref_fit_free(hd)
        # plain-C restatement: one call
        cap = C.c_size_t()
        self._call("fit_capacity", C.c_int(w), C.c_int(h), C.byref(c), C.c_size_t(init.size() if init else 0),
                   C.byref(cap))
        out = SiteStore(0)
        sv, keep = out._view(capacity=int(cap.value))
        f = CandidateField()
        f.resize(w, h, cfg.k)
        fv = f._view()
        hist = (_abi.HistoryRowC * max(cfg.iters, 1))()
        sc = C.c_double()
        iv = None
        if init is not None:
            iv, ikeep = init._view()
        self._call("fit", _ptr(target.data), C.c_int(w), C.c_int(h), C.byref(c), _ref(iv), _ref(sv), _ref(fv),
                   hist, C.byref(sc))
        out._absorb(sv, keep)
        f._absorb(fv)
        rows = [HistoryRow(r.iter, r.loss, r.psnr, r.active_sites, r.ms) for r in hist[: cfg.iters]]
        return FitResult(out, f, rows, float(sc.value))


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
        _cache[key] = OracleBackend(lib, "sadref_", "ref", threads=threads)
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
        _cache["c"] = OracleBackend(lib, "sado_", "c")
    return _cache["c"]


def build(verbose: bool = False) -> None:
    """Compile libsado.so always and libsadref.so when /root/reference is present."""
    import subprocess
    subprocess.run(["make", "-s", "-f", os.path.join(HERE, "Makefile")], check=True,
                   stdout=None if verbose else subprocess.DEVNULL)
