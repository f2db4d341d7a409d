"""Python mirror of the reference `sad::` API (candidates.hpp, render.hpp, grad.hpp, train.hpp,
budget.hpp) over a C-ABI library with the entry points of include/sad_b200.h.

`Backend` binds one library.  The product binding (`gpu_backend()`) loads the in-tree CUDA
library `libsad_b200.so` and fails loudly when it is missing or when no GPU is present — there is
no CPU fallback on the product path.  The same class is reused by the test-only oracle bindings
(oracle/bindings.py) so parity tests can call the reference and the GPU with identical code.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from typing import List, Optional, Sequence

import numpy as np

from . import _abi
from .types import (AdamState, CandidateField, FitResult, GradBuffer, HistoryRow, ImageBuffer, PassSpec,
                    RefreshMode, RunOpts, SiteStore, StatsResult, Stencil, TrainConfig, normalization_scale,
                    psnr_from_loss)


class SadError(Exception):
    code = -1


class InvalidArgument(SadError, ValueError):
    """std::invalid_argument (bad input, stale field, empty candidate list)."""


class StaleField(InvalidArgument):
    code = _abi.SAD_ESTALE


class EmptyList(InvalidArgument):
    code = _abi.SAD_EEMPTY


class NumericError(SadError, ArithmeticError):
    """sad::numeric_error (types.hpp:14-17)."""
    code = _abi.SAD_ENUMERIC


class FormatError(SadError):
    code = _abi.SAD_EFORMAT


class CudaError(SadError, RuntimeError):
    code = _abi.SAD_ECUDA


class CapacityError(SadError, MemoryError):
    code = _abi.SAD_ENOMEM


_EXC = {
    _abi.SAD_EINVAL: InvalidArgument,
    _abi.SAD_ESTALE: StaleField,
    _abi.SAD_EEMPTY: EmptyList,
    _abi.SAD_ENUMERIC: NumericError,
    _abi.SAD_EFORMAT: FormatError,
    _abi.SAD_ECUDA: CudaError,
    _abi.SAD_ENOMEM: CapacityError,
}

_P = C.c_void_p
_dp = C.POINTER(C.c_double)


def _ref(x):
    """byref, or NULL for a resident object (its views are None)."""
    return None if x is None else C.byref(x)


def _ptr(a: np.ndarray, t=C.c_double):
    return a.ctypes.data_as(C.POINTER(t))


class Backend:
    """The C-ABI binding of include/sad_b200.h (`sad_` prefix, context-first calls).

    Test-only oracle bindings (oracle/bindings.py) subclass it and override the few hooks below
    (`_pre`, `_thr`, `_fit`, `decode_render`) for the CPU libraries' argument conventions; the product
    package itself knows nothing about them."""

    def __init__(self, lib: C.CDLL, prefix: str = "sad_", ctx=None):
        self.lib = lib
        self.prefix = prefix
        self.ctx = ctx
        self.lib.__getattr__(prefix + "last_error").restype = C.c_char_p

    # ------------------------------------------------------------------ plumbing
    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def _pre(self, name):
        """Leading arguments of a call: the context handle, except for context-free entry points."""
        return () if name in _NO_CTX else (self.ctx,)

    def _call(self, name, *args):
        rc = self._fn(name)(*self._pre(name), *args)
        if rc != 0:
            msg = self._fn("last_error")().decode(errors="replace")
            raise _EXC.get(rc, SadError)(f"{self.prefix}{name}: {msg}")

    def _thr(self):
        """Trailing worker-count arguments (none: RunOpts.threads is ignored on the device)."""
        return ()

    # ------------------------------------------------------------------ device-resident objects
    def sites_alloc(self, capacity: int) -> "ResidentSites":
        self._call("sites_alloc", C.c_size_t(capacity))
        return ResidentSites(self)

    def sites_upload(self, sites: SiteStore, capacity: Optional[int] = None) -> "ResidentSites":
        """Upload into the context's resident store, with room for `capacity` sites (densify appends)."""
        sv, keep = sites._view(capacity=capacity)
        self._call("sites_upload", _ref(sv))
        return ResidentSites(self)

    def sites_download(self) -> SiteStore:
        n, cap, gen = self._sites_info()
        out = SiteStore(0)
        sv, keep = out._view(capacity=max(n, 1))
        self._call("sites_download", _ref(sv))
        out._absorb(sv, keep)
        return out

    def _sites_info(self):
        n, cap, gen = C.c_size_t(), C.c_size_t(), C.c_uint64()
        self._call("sites_info", C.byref(n), C.byref(cap), C.byref(gen))
        return n.value, cap.value, gen.value

    def field_alloc(self, width: int, height: int, k: int, cell: int = 1) -> "ResidentField":
        self._call("field_alloc", C.c_int(width), C.c_int(height), C.c_int(k), C.c_int(cell))
        return ResidentField(self)

    def field_upload(self, field: CandidateField) -> "ResidentField":
        fv = field._view()
        self._call("field_upload", _ref(fv))
        return ResidentField(self)

    def field_download(self) -> CandidateField:
        m = self._field_meta()
        f = CandidateField()
        f.resize(m.width, m.height, m.k, m.cell)
        fv = f._view()
        self._call("field_download", _ref(fv))
        f._absorb(fv)
        return f

    def _field_meta(self):
        fv = _abi.FieldView()
        fv.ids = None
        self._call("field_download", C.byref(fv))
        return fv

    # ------------------------------------------------------------------ candidates.hpp
    def jump_step(self, t: int, b: int) -> int:
        out = C.c_uint32()
        self._call("jump_step", C.c_uint32(t), C.c_uint32(b), C.byref(out))
        return out.value

    def full_refresh_passes(self, gw, gh, extra_step1) -> List[PassSpec]:
        buf = (_abi.PassSpec * (64 + max(extra_step1, 0)))()
        n = C.c_int(len(buf))
        self._call("full_refresh_passes", C.c_int(gw), C.c_int(gh), C.c_int(extra_step1), buf, C.byref(n))
        return [PassSpec(buf[i].step, Stencil(buf[i].stencil)) for i in range(n.value)]

    def schedule_passes(self, gw, gh, total) -> List[PassSpec]:
        """schedule_passes (candidates.cpp:50-62): `total` passes of the jump schedule, Box3 floods at
        halving steps then Axial step-1 passes."""
        buf = (_abi.PassSpec * max(total, 1))()
        n = C.c_int(len(buf))
        self._call("schedule_passes", C.c_int(gw), C.c_int(gh), C.c_int(total), buf, C.byref(n))
        return [PassSpec(buf[i].step, Stencil(buf[i].stencil)) for i in range(n.value)]

    def jfa_seed(self, sites: SiteStore, field: CandidateField):
        sv, keep = sites._view()
        fv = field._view()
        self._call("jfa_seed", _ref(sv), _ref(fv))
        field._absorb(fv)

    def run_passes(self, sites: SiteStore, field: CandidateField, seq: Sequence[PassSpec], inject: int,
                   seed: int, opts: RunOpts = RunOpts()):
        sv, keep = sites._view()
        fv = field._view()
        arr = (_abi.PassSpec * max(len(seq), 1))(*[_abi.PassSpec(p.step, int(p.stencil)) for p in seq])
        self._call("run_passes", _ref(sv), _ref(fv), arr, C.c_int(len(seq)), C.c_int(inject),
                   C.c_uint64(seed), C.c_int(int(opts.fp64)), *self._thr())
        field._absorb(fv)

    def propagate_pass(self, sites, field, p: PassSpec, inject, seed, opts: RunOpts = RunOpts()):
        self.run_passes(sites, field, [p], inject, seed, opts)

    def refresh(self, sites: SiteStore, field: CandidateField, mode: RefreshMode, passes: int, inject: int,
                seed: int, opts: RunOpts = RunOpts()):
        sv, keep = sites._view()
        fv = field._view()
        self._call("refresh", _ref(sv), _ref(fv), C.c_int(int(mode)), C.c_int(passes), C.c_int(inject),
                   C.c_uint64(seed), C.c_int(int(opts.fp64)), *self._thr())
        field._absorb(fv)

    def exact_topk_batch(self, sites: SiteStore, pixels, k: int, scale: float, fp64: bool = True) -> np.ndarray:
        xy = np.ascontiguousarray(np.asarray(pixels, np.int32).reshape(-1, 2))
        out = np.full(xy.shape[0] * k, _abi.EMPTY_ID, np.uint32)
        sv, keep = sites._view()
        self._call("exact_topk_batch", _ref(sv), _ptr(xy, C.c_int32), C.c_size_t(xy.shape[0]), C.c_int(k),
                   C.c_double(scale), C.c_int(int(fp64)), _ptr(out, C.c_uint32))
        return out.reshape(-1, k)

    # ------------------------------------------------------------------ render.hpp
    def render_image(self, sites: SiteStore, field: CandidateField, opts: RunOpts = RunOpts()) -> ImageBuffer:
        out = ImageBuffer(field.width, field.height)
        sv, keep = sites._view()
        fv = field._view()
        self._call("render_image", _ref(sv), _ref(fv), C.c_int(int(opts.fp64)), *self._thr(), _ptr(out.data))
        return out

    def pixel_weights_batch(self, sites, field, pixels):
        xy = np.ascontiguousarray(np.asarray(pixels, np.int32).reshape(-1, 2))
        q = xy.shape[0]
        ids = np.zeros(q * 16, np.uint32)
        w = np.zeros(q * 16, np.float64)
        n = np.zeros(q, np.int32)
        sv, keep = sites._view()
        fv = field._view()
        self._call("pixel_weights", _ref(sv), _ref(fv), _ptr(xy, C.c_int32), C.c_size_t(q),
                   _ptr(ids, C.c_uint32), _ptr(w), _ptr(n, C.c_int32))
        return ids.reshape(q, 16), w.reshape(q, 16), n

    def pixel_weights(self, sites, field, px, py):
        ids, w, n = self.pixel_weights_batch(sites, field, [(px, py)])
        return ids[0, : n[0]].copy(), w[0, : n[0]].copy()

    def render_id_map(self, sites, field, opts: RunOpts = RunOpts()) -> np.ndarray:
        out = np.zeros(field.width * field.height, np.uint32)
        sv, keep = sites._view()
        fv = field._view()
        self._call("render_id_map", _ref(sv), _ref(fv), _ptr(out, C.c_uint32))
        return out

    # ------------------------------------------------------------------ grad.hpp
    def backward_image(self, sites, field, target: ImageBuffer, out: GradBuffer, opts: RunOpts = RunOpts(),
                       with_removal: bool = True) -> float:
        if target.width != field.width or target.height != field.height:
            raise InvalidArgument("backward: target size mismatch")
        out.resize(sites.size())
        g = np.zeros(max(sites.size(), 1) * 11, np.float64)
        nf = C.c_uint64()
        loss = C.c_double()
        sv, keep = sites._view()
        fv = field._view()
        self._call("backward_image", _ref(sv), _ref(fv), _ptr(target.data), C.c_int(int(opts.fp64)),
                   C.c_int(int(with_removal)), *self._thr(), _ptr(g), C.byref(nf), C.byref(loss))
        out.data = g[: sites.size() * 11].reshape(-1, 11).copy()
        out.nonfinite = int(nf.value)
        return float(loss.value)

    def image_loss(self, sites, field, target: ImageBuffer, opts: RunOpts = RunOpts()) -> float:
        if target.width != field.width or target.height != field.height:
            raise InvalidArgument("loss: target size mismatch")
        loss = C.c_double()
        sv, keep = sites._view()
        fv = field._view()
        self._call("image_loss", _ref(sv), _ref(fv), _ptr(target.data), C.c_int(int(opts.fp64)),
                   C.byref(loss))
        return float(loss.value)

    def backward_pixel_grad(self, sites, field, dl: ImageBuffer, out: GradBuffer, opts: RunOpts = RunOpts()):
        out.resize(sites.size())
        g = np.zeros(max(sites.size(), 1) * 11, np.float64)
        nf = C.c_uint64()
        sv, keep = sites._view()
        fv = field._view()
        self._call("backward_pixel_grad", _ref(sv), _ref(fv), _ptr(dl.data), C.c_int(dl.width), C.c_int(dl.height),
                   C.c_int(int(opts.fp64)), _ptr(g), C.byref(nf))
        out.data = g[: sites.size() * 11].reshape(-1, 11).copy()
        out.nonfinite = int(nf.value)

    # ------------------------------------------------------------------ train.hpp
    def adam_step(self, sites: SiteStore, g: GradBuffer, adam: AdamState, width, height, cfg: TrainConfig):
        if g.size() != sites.size():
            raise InvalidArgument("adam_step: gradient size mismatch")
        sv, keep = sites._view()
        av, akeep = adam._view(sites.size())
        gd = np.ascontiguousarray(g.data.reshape(-1))
        if gd.size == 0:
            gd = np.zeros(11)
        c = cfg.to_c()
        self._call("adam_step", _ref(sv), _ptr(gd), C.byref(av), C.c_int(width), C.c_int(height), C.byref(c))
        sites._absorb(sv, keep)
        adam._absorb(av, akeep)

    def tau_diffusion(self, sites: SiteStore, field: CandidateField, lam: float, g: GradBuffer,
                      opts: RunOpts = RunOpts()):
        """tau_diffusion (train.hpp:43-44, train.cpp:171-213): mixes each pixel owner's logtau gradient
        with the mean over its co-candidates; other channels and non-owners are untouched."""
        if lam == 0:
            return
        if lam < 0 or lam > 1:
            raise InvalidArgument("tau_diffusion: lambda out of [0,1]")
        if g.size() != sites.size():
            raise InvalidArgument("tau_diffusion: size mismatch")
        sv, keep = sites._view()
        fv = field._view()
        gd = np.ascontiguousarray(g.data, dtype=np.float64).reshape(-1).copy()
        if gd.size == 0:
            gd = np.zeros(11)
        self._call("tau_diffusion", _ref(sv), _ref(fv), C.c_double(lam), _ptr(gd))
        g.data = gd[: sites.size() * 11].reshape(-1, 11).copy()

    def clamp_project(self, sites: SiteStore, width, height, cfg: TrainConfig):
        sv, keep = sites._view()
        c = cfg.to_c()
        self._call("clamp_project", _ref(sv), C.c_int(width), C.c_int(height), C.byref(c))
        sites._absorb(sv, keep)

    def init_sites(self, sites: SiteStore, target: ImageBuffer, n: int, cfg: TrainConfig):
        tmp = SiteStore(0)
        sv, keep = tmp._view(capacity=max(n, 1))
        c = cfg.to_c()
        self._call("init_sites", _ref(sv), _ptr(target.data), C.c_int(target.width), C.c_int(target.height),
                   C.c_int(n), C.byref(c))
        gen = sites.generation
        sites._absorb(sv, keep)
        sites.generation = gen + 1 + n

    # ------------------------------------------------------------------ budget.hpp
    def accumulate_stats(self, sites, field, target: ImageBuffer, opts: RunOpts = RunOpts()) -> StatsResult:
        if target.width != field.width or target.height != field.height:
            raise InvalidArgument("stats: target size mismatch")
        r = StatsResult(sites.size())
        buf = np.zeros(max(sites.size(), 1) * 8, np.float64)
        valid = C.c_uint64()
        sv, keep = sites._view()
        fv = field._view()
        self._call("accumulate_stats", _ref(sv), _ref(fv), _ptr(target.data), *self._thr(), _ptr(buf),
                   C.byref(valid))
        r.data = buf[: sites.size() * 8].reshape(-1, 8).copy()
        r.valid_pixels = int(valid.value)
        return r

    def prune(self, sites: SiteStore, stats: StatsResult, percentile: float) -> int:
        if stats.data.shape[0] != sites.size():
            raise InvalidArgument("prune: stats size mismatch")
        sv, keep = sites._view()
        sd = np.ascontiguousarray(stats.data.reshape(-1)) if stats.data.size else np.zeros(8)
        n = C.c_int()
        self._call("prune", _ref(sv), _ptr(sd), C.c_uint64(stats.valid_pixels), C.c_double(percentile),
                   C.byref(n))
        sites._absorb(sv, keep)
        return n.value

    def densify(self, sites: SiteStore, adam: AdamState, stats: StatsResult, target: ImageBuffer, percentile: float,
                cfg: TrainConfig) -> int:
        if stats.data.shape[0] != sites.size():
            raise InvalidArgument("densify: stats size mismatch")
        cap = 2 * sites.size() + 1
        sv, keep = sites._view(capacity=cap)
        av, akeep = adam._view(cap)
        sd = np.ascontiguousarray(stats.data.reshape(-1)) if stats.data.size else np.zeros(8)
        c = cfg.to_c()
        n = C.c_int()
        self._call("densify", _ref(sv), C.byref(av), _ptr(sd), _ptr(target.data), C.c_int(target.width),
                   C.c_int(target.height), C.c_double(percentile), C.byref(c), C.byref(n))
        sites._absorb(sv, keep)
        adam._absorb(av, akeep)
        return n.value

    def bpp_target_count(self, bpp, width, height) -> int:
        out = C.c_uint64()
        self._call("bpp_target_count", C.c_double(bpp), C.c_int(width), C.c_int(height), C.byref(out))
        return out.value

    def simulate_schedule(self, n0, scale, cfg: TrainConfig) -> int:
        out = C.c_int()
        c = cfg.to_c()
        self._call("simulate_schedule", C.c_int(n0), C.c_double(scale), C.byref(c), C.byref(out))
        return out.value

    def plan_schedule(self, n0, target, cfg: TrainConfig) -> float:
        out = C.c_double()
        c = cfg.to_c()
        self._call("plan_schedule", C.c_int(n0), C.c_uint64(target), C.byref(c), C.byref(out))
        return out.value

    # ------------------------------------------------------------------ codec.hpp (decode path)
    def encode_sites(self, sites: SiteStore, width: int, height: int) -> bytes:
        """write_file (codec.cpp:147-177) into memory: the `.sad` container bytes."""
        sv, keep = sites._view()
        n = C.c_size_t()
        self._call("encode", _ref(sv), C.c_int(width), C.c_int(height), None, C.c_size_t(0), C.byref(n))
        buf = (C.c_uint8 * n.value)()
        self._call("encode", _ref(sv), C.c_int(width), C.c_int(height), buf, C.c_size_t(n.value), C.byref(n))
        return bytes(buf)

    def decode_sites(self, data: bytes):
        """read_file (codec.cpp:179-222): returns (width, height, SiteStore)."""
        count = max((len(data) - 58) // 16, 0) if len(data) >= 58 else 0
        st = SiteStore(0)
        sv, keep = st._view(capacity=count + 1)
        buf = (C.c_uint8 * len(data)).from_buffer_copy(data)
        w, h = C.c_int(), C.c_int()
        self._call("decode", buf, C.c_size_t(len(data)), _ref(sv), C.byref(w), C.byref(h))
        st._absorb(sv, keep)
        return w.value, h.value, st

    def write_file(self, path: str, sites: SiteStore, width: int, height: int):
        with open(path, "wb") as f:
            f.write(self.encode_sites(sites, width, height))

    def read_file(self, path: str):
        with open(path, "rb") as f:
            return self.decode_sites(f.read())

    def decode_render(self, data: bytes, k: int = 8, passes: int = 16, inject: int = 4, seed: int = 1,
                      fp64: bool = False):
        """Decode pipeline on the device: bytes -> sites -> refresh(Full, passes) -> render_image.
        Returns (ImageBuffer, SiteStore)."""
        buf = (C.c_uint8 * len(data)).from_buffer_copy(data)
        w, h, cnt = C.c_int(), C.c_int(), C.c_uint32()
        self._call("decode_header", buf, C.c_size_t(len(data)), C.byref(w), C.byref(h), C.byref(cnt))
        img = ImageBuffer(w.value, h.value)
        st = SiteStore(0)
        sv, keep = st._view(capacity=cnt.value + 1)
        self._call("decode_render", buf, C.c_size_t(len(data)), C.c_int(k), C.c_int(passes), C.c_int(inject),
                   C.c_uint64(seed), C.c_int(int(fp64)), _ptr(img.data), _ref(sv))
        st._absorb(sv, keep)
        return img, st

    # ------------------------------------------------------------------ fit (train.cpp:221-311)
    def fit(self, target: ImageBuffer, cfg: TrainConfig) -> FitResult:
        return self._fit(target, cfg, None)

    def fit_store(self, sites: SiteStore, target: ImageBuffer, cfg: TrainConfig) -> FitResult:
        return self._fit(target, cfg, sites)

    def _collect_run(self, run, w, h, cfg) -> FitResult:
        n, nh, sc = C.c_size_t(), C.c_int(), C.c_double()
        self._call("fit_info", run, C.byref(n), C.byref(nh), C.byref(sc))
        res = self._fit_collect(w, h, cfg, int(n.value), int(nh.value), float(sc.value),
                                lambda sv, fv, hist: self._call("fit_download", run, sv, fv, hist))
        tot = C.c_double()
        ph = (C.c_double * 8)()
        self._call("fit_timing", run, C.byref(tot), ph)
        res.timing = {"total_ms": tot.value}  # device time of the fit loop (refreshes included)
        return res

    def fit_strips_loopback(self, target: ImageBuffer, cfg: TrainConfig, world: int) -> List[FitResult]:
        """Row-strip fit (config 5 partition) with `world` virtual ranks on this device; returns every
        rank's result (all equal to fit() when the partition is exact)."""
        c = cfg.to_c()
        w, h = target.width, target.height
        runs = []
        try:
            for _ in range(world):
                run = C.c_void_p()
                self._call("fit_create", C.c_int(w), C.c_int(h), C.byref(c), C.byref(run))
                runs.append(run)
                self._call("fit_set_target", run, _ptr(target.data))
            arr = (C.c_void_p * world)(*[r.value for r in runs])
            self._call("fit_run_strips_loopback", arr, C.c_int(world))
            out = []
            for r in runs:
                res = self._collect_run(r, w, h, cfg)
                sent = C.c_longlong()
                self._call("fit_strip_exchange", r, C.byref(sent))
                res.timing["records_sent"] = sent.value
                out.append(res)
            return out
        finally:
            for r in runs:
                self.lib.sad_fit_destroy(r)

    def strip_comm(self, rank: int, world: int, nccl_id: bytes):
        """NCCL communicator over the strip ranks (one per process; NCCL ids are single-use)."""
        comm = C.c_void_p()
        idb = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
        self._call("strip_comm_create", C.c_int(rank), C.c_int(world), idb, C.byref(comm))
        return comm

    def fit_strips(self, target: ImageBuffer, cfg: TrainConfig, comm, init: Optional[SiteStore] = None) -> FitResult:
        """This rank's part of a row-strip multi-GPU fit over NCCL (one process per GPU)."""
        c = cfg.to_c()
        w, h = target.width, target.height
        run = C.c_void_p()
        self._call("fit_create", C.c_int(w), C.c_int(h), C.byref(c), C.byref(run))
        try:
            self._call("fit_set_target", run, _ptr(target.data))
            sv = None
            if init is not None:
                sv, keep = init._view()
            self._call("fit_run_strips", run, getattr(comm, "handle", comm), _ref(sv))
            res = self._collect_run(run, w, h, cfg)
            sent = C.c_longlong()
            self._call("fit_strip_exchange", run, C.byref(sent))
            res.timing["records_sent"] = sent.value
            return res
        finally:
            self.lib.sad_fit_destroy(run)

    def strip_comm_host(self, group=None) -> "HostStripComm":
        """A host-staged strip communicator over a torch.distributed process group (e.g. gloo): the
        library copies device data to pinned host memory and calls back into Python for each collective,
        so several processes can share one GPU (tests) or GPUs without NCCL can take part."""
        return HostStripComm(self, group)

    def nccl_unique_id(self) -> bytes:
        buf = (C.c_uint8 * 128)()
        self._call("nccl_unique_id", buf)
        return bytes(buf)

    def fit_oneshot(self, target: ImageBuffer, cfg: TrainConfig, init: Optional[SiteStore] = None) -> FitResult:
        """sad_fit / sad_fit_store: the single C call an FFI binding would make (no cached run)."""
        c = cfg.to_c()
        cap = C.c_size_t()
        self._call("fit_capacity", C.c_int(target.width), C.c_int(target.height), C.byref(c),
                   C.c_size_t(init.size() if init is not None else 0), C.byref(cap))
        sc = C.c_double()
        n_hist = max(cfg.iters, 1)

        def run(sv, fv, hist):
            if init is None:
                self._call("fit", _ptr(target.data), C.c_int(target.width), C.c_int(target.height), C.byref(c),
                           sv, fv, hist, C.byref(sc))
            else:
                iv, ikeep = init._view()
                self._call("fit_store", _ptr(target.data), C.c_int(target.width), C.c_int(target.height),
                           _ref(iv), C.byref(c), sv, fv, hist, C.byref(sc))

        st = SiteStore(0)
        sv, keep = st._view(capacity=max(int(cap.value), 1))
        f = CandidateField()
        f.resize(target.width, target.height, cfg.k)
        fv = f._view()
        hist = (_abi.HistoryRowC * n_hist)()
        run(_ref(sv), _ref(fv), hist)
        st._absorb(sv, keep)
        f._absorb(fv)
        rows = [HistoryRow(r.iter, r.loss, r.psnr, r.active_sites, r.ms) for r in hist[:cfg.iters]]
        return FitResult(st, f, rows, sc.value)

    def _fit_run(self, w, h, c):
        """Resident fit runs are cached per (shape, config): repeated fits reuse the device workspace
        (sites, field, record pools, graphs) instead of reallocating ~hundreds of MB per call."""
        if not hasattr(self, "_runs"):
            self._runs = {}
        key = (w, h, bytes(c))
        run = self._runs.get(key)
        if run is None:
            while len(self._runs) >= 2:
                _, old = self._runs.popitem()
                self.lib.sad_fit_destroy(old)
            run = _P()
            self._call("fit_create", C.c_int(w), C.c_int(h), C.byref(c), C.byref(run))
            self._runs[key] = run
        return run

    def close(self):
        for run in getattr(self, "_runs", {}).values():
            self.lib.sad_fit_destroy(run)
        self._runs = {}

    def _fit(self, target: ImageBuffer, cfg: TrainConfig, init: Optional[SiteStore]) -> FitResult:
        c = cfg.to_c()
        w, h = target.width, target.height
        run = self._fit_run(w, h, c)
        self._call("fit_set_target", run, _ptr(target.data))
        if init is None:
            self._call("fit_run_init", run)
        else:
            sv, keep = init._view()
            self._call("fit_run_store", run, _ref(sv))
        n = C.c_size_t()
        nh = C.c_int()
        sc = C.c_double()
        self._call("fit_info", run, C.byref(n), C.byref(nh), C.byref(sc))
        res = self._fit_collect(w, h, cfg, int(n.value), int(nh.value), float(sc.value),
                                lambda sv, fv, hist: self._call("fit_download", run, sv, fv, hist))
        tot = C.c_double()
        ph = (C.c_double * 8)()
        self._call("fit_timing", run, C.byref(tot), ph)
        res.timing = {"total_ms": tot.value, "propagate_ms": ph[0], "fwd_bwd_ms": ph[1],
                      "adam_ms": ph[2], "events_ms": ph[3]}
        return res

    def _fit_collect(self, w, h, cfg, n, nh, sc, download) -> FitResult:
        st = SiteStore(0)
        sv, keep = st._view(capacity=max(n, 1))
        f = CandidateField()
        f.resize(w, h, cfg.k)
        fv = f._view()
        hist = (_abi.HistoryRowC * max(nh, 1))()
        download(_ref(sv), _ref(fv), hist)
        sv.size = n
        st._absorb(sv, keep)
        f._absorb(fv)
        rows = [HistoryRow(r.iter, r.loss, r.psnr, r.active_sites, r.ms) for r in hist[:nh]]
        return FitResult(st, f, rows, sc)


_AG_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t)
_EX_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_void_p), C.POINTER(C.c_size_t),
                     C.POINTER(C.c_void_p), C.POINTER(C.c_size_t))


class HostStripComm:
    """sad_strip_comm_create_host over a torch.distributed group: all-gather and grouped point-to-point
    transfers of host byte buffers (include/sad_b200.h).  Pass `.handle` to Backend.fit_strips."""

    def __init__(self, backend: "Backend", group=None):
        import torch
        import torch.distributed as dist
        self._B = backend
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        world = self.world

        def _host(ptr, n):
            return torch.frombuffer((C.c_uint8 * n).from_address(ptr), dtype=torch.uint8).clone()

        def allgather(user, send, recv, nbytes):
            try:
                mine = _host(send, nbytes) if nbytes else torch.empty(0, dtype=torch.uint8)
                outs = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(world)]
                dist.all_gather(outs, mine, group=group)
                for q, t in enumerate(outs):
                    if nbytes:
                        C.memmove(recv + q * nbytes, t.data_ptr(), nbytes)
                return 0
            except Exception:  # noqa: BLE001 - reported to the library as a failed collective
                import traceback
                traceback.print_exc()
                return 1

        def exchange(user, n, peer, send, sbytes, recv, rbytes):
            try:
                reqs, outs = [], []
                for i in range(n):
                    if sbytes[i]:
                        t = _host(send[i], sbytes[i])
                        reqs.append((dist.isend(t, int(peer[i]), group=group), t))
                    if rbytes[i]:
                        t = torch.empty(rbytes[i], dtype=torch.uint8)
                        reqs.append((dist.irecv(t, int(peer[i]), group=group), t))
                        outs.append((recv[i], t))
                for r, _ in reqs:
                    r.wait()
                for ptr, t in outs:
                    C.memmove(ptr, t.data_ptr(), t.numel())
                return 0
            except Exception:  # noqa: BLE001
                import traceback
                traceback.print_exc()
                return 1

        self._ag = _AG_FN(allgather)
        self._ex = _EX_FN(exchange)
        self.handle = C.c_void_p()
        backend._call("strip_comm_create_host", C.c_int(self.rank), C.c_int(world), self._ag, self._ex, None,
                      C.byref(self.handle))

    def close(self):
        if self.handle:
            self._B.lib.sad_strip_comm_destroy(self.handle)
            self.handle = C.c_void_p()


_NO_CTX = {"jump_step", "full_refresh_passes", "schedule_passes", "bpp_target_count", "simulate_schedule",
           "plan_schedule", "fit_set_target", "fit_set_target_device", "fit_run_init", "fit_run_store",
           "fit_info", "fit_download", "fit_render_device", "fit_timing", "fit_bench", "fit_set_profiling",
           "fit_point_query", "fit_capacity", "fit_run_strips", "fit_run_strips_loopback", "nccl_unique_id", "strip_comm_create",
           "strip_comm_create_host", "fit_strip_exchange", "encode", "decode", "decode_header", "bpp",
           "last_error"}

# ---------------------------------------------------------------------- product binding
_HERE = os.path.dirname(os.path.abspath(__file__))
# SAD_LIB selects another build of the same sources (tests: the bound-checked libsad_b200_checked.so)
LIB_PATH = os.environ.get("SAD_LIB") or os.path.join(_HERE, "libsad_b200.so")
_lock = threading.Lock()
_gpu = None


def load_library(path: Optional[str] = None) -> C.CDLL:
    path = path or LIB_PATH
    if not os.path.exists(path):
        raise ImportError(f"CUDA library {path} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    lib.sad_last_error.restype = C.c_char_p
    lib.sad_ctx_launch_count.restype = C.c_uint64
    lib.sad_ctx_launch_count.argtypes = [_P]
    lib.sad_debug_check_failures.restype = C.c_longlong
    lib.sad_fit_destroy.argtypes = [_P]
    lib.sad_strip_comm_destroy.argtypes = [_P]
    lib.sad_ctx_destroy.argtypes = [_P]
    return lib


def gpu_backend(device: int = 0) -> Backend:
    """The product backend (CUDA, sm_100a).  Raises if the extension or the GPU is unavailable."""
    global _gpu
    with _lock:
        if _gpu is None:
            lib = load_library()
            ctx = _P()
            rc = lib.sad_ctx_create(C.c_int(device), None, C.byref(ctx))
            if rc != 0:
                raise CudaError("sad_ctx_create: " + lib.sad_last_error().decode(errors="replace"))
            _gpu = Backend(lib, "sad_", ctx=ctx)
        return _gpu


class ResidentSites:
    """The context's device-resident SiteStore (sad_sites_alloc / sad_sites_upload): pass it
    wherever a SiteStore is expected to run on the device copy without host transfers."""

    def __init__(self, backend: "Backend"):
        self._B = backend

    def _view(self, capacity=None):
        return None, None

    def _absorb(self, v, bufs):
        pass

    def size(self) -> int:
        return self._B._sites_info()[0]

    @property
    def generation(self) -> int:
        return self._B._sites_info()[2]


class ResidentField:
    """The context's device-resident CandidateField (sad_field_alloc / sad_field_upload)."""

    def __init__(self, backend: "Backend"):
        self._B = backend

    def _view(self):
        return None

    def _absorb(self, v):
        pass

    def __getattr__(self, name):
        if name in ("width", "height", "cell", "gw", "gh", "k", "synced_generation", "refresh_count",
                    "pass_index"):
            return getattr(self._B._field_meta(), name)
        raise AttributeError(name)
