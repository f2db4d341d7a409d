"""Host-side value types mirroring the reference's `sad::` types (types.hpp, grad.hpp, train.hpp,
budget.hpp).  They own numpy storage with the reference's exact layouts so buffers cross the C ABI
without conversion:

* SiteStore      — types.hpp:37-63   (ten double SoA arrays + u8 active/frozen + generation)
* CandidateField — types.hpp:84-110  (u32 ids[(gy*gw+gx)*k+i], sentinel 0xffffffff)
* ImageBuffer    — types.hpp:67-79   (interleaved RGB doubles, row-major)
* GradBuffer     — grad.hpp:35-57    (n x 11 doubles: 10 gradient slots + removal delta)
* AdamState      — train.hpp:13-21   (m, v: n x 10 doubles, global step t)
* StatsResult    — budget.hpp:14-25  (n x 8 doubles + valid_pixels)
* TrainConfig    — types.hpp:112-167 (field for field)
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _abi

EMPTY = _abi.EMPTY_ID

# GradSlot (grad.hpp:13-26)
kGradX, kGradY, kGradLogTau, kGradRadius, kGradColR, kGradColG, kGradColB, kGradDirX, kGradDirY, kGradAniso = range(10)
kGradSlots = 10
kChannels = 11
kRemovalSaturated = 1e6

_PARAMS = ("x", "y", "log_tau", "radius", "col_r", "col_g", "col_b", "dir_x", "dir_y", "aniso")


class Stencil(enum.IntEnum):
    Axial = 0
    Box3 = 1


class RefreshMode(enum.IntEnum):
    Full = 0
    WarmStart = 1


@dataclass
class PassSpec:
    step: int = 1
    stencil: Stencil = Stencil.Axial


@dataclass
class RunOpts:
    """RunOpts (types.hpp:170-175).  `threads` is accepted and ignored by the GPU backend."""
    fp64: bool = True
    threads: int = 1


@dataclass
class Site:
    """Site (types.hpp:22-31)."""
    x: float = 0.0
    y: float = 0.0
    log_tau: float = 7.5
    radius: float = 1.0
    color: tuple = (0.0, 0.0, 0.0)
    dir: tuple = (1.0, 0.0)
    aniso: float = 0.0
    active: bool = True
    frozen: bool = False


class SiteStore:
    """SiteStore (types.hpp:37-63).  Slots are never erased; deactivate() parks at (-1,-1)."""

    def __init__(self, n: int = 0):
        self.generation = 0
        self._alloc(n)

    def _alloc(self, n):
        for p in _PARAMS:
            setattr(self, p, np.zeros(n, np.float64))
        self.dir_x[:] = 1.0
        self.active = np.zeros(n, np.uint8)
        self.frozen = np.zeros(n, np.uint8)

    # --- reference methods (types.cpp:7-80)
    def size(self) -> int:
        return int(self.x.shape[0])

    def clear(self):
        self._alloc(0)
        self.bump()

    def resize(self, n: int):
        old = self.size()
        for p in _PARAMS:
            a = getattr(self, p)
            b = np.zeros(n, np.float64)
            if p == "dir_x":
                b[:] = 1.0
            b[: min(old, n)] = a[: min(old, n)]
            setattr(self, p, b)
        for p in ("active", "frozen"):
            a = getattr(self, p)
            b = np.zeros(n, np.uint8)
            b[: min(old, n)] = a[: min(old, n)]
            setattr(self, p, b)
        self.bump()

    def append(self, s: Site) -> int:
        i = self.size()
        self.resize(i + 1)
        self.generation -= 1  # resize bumped; set() below bumps once like append()
        self.set(i, s)
        return i

    def get(self, i: int) -> Site:
        return Site(float(self.x[i]), float(self.y[i]), float(self.log_tau[i]), float(self.radius[i]),
                    (float(self.col_r[i]), float(self.col_g[i]), float(self.col_b[i])),
                    (float(self.dir_x[i]), float(self.dir_y[i])), float(self.aniso[i]),
                    bool(self.active[i]), bool(self.frozen[i]))

    def set(self, i: int, s: Site):
        self.x[i], self.y[i], self.log_tau[i], self.radius[i] = s.x, s.y, s.log_tau, s.radius
        self.col_r[i], self.col_g[i], self.col_b[i] = s.color
        self.dir_x[i], self.dir_y[i] = s.dir
        self.aniso[i] = s.aniso
        self.active[i] = 1 if s.active else 0
        self.frozen[i] = 1 if s.frozen else 0
        self.bump()

    def deactivate(self, i: int):
        self.active[i] = 0
        self.x[i] = -1.0
        self.y[i] = -1.0
        self.bump()

    def bump(self):
        self.generation += 1

    def active_ids(self) -> np.ndarray:
        return np.nonzero(self.active)[0].astype(np.uint32)

    def active_count(self) -> int:
        return int(np.count_nonzero(self.active))

    def copy(self) -> "SiteStore":
        o = SiteStore(0)
        for p in _PARAMS + ("active", "frozen"):
            setattr(o, p, getattr(self, p).copy())
        o.generation = self.generation
        return o

    # --- ABI view.  `capacity` > size leaves room for densify appends.
    def _view(self, capacity: Optional[int] = None):
        n = self.size()
        cap = max(n, capacity or n, 1)
        bufs = {}
        for p in _PARAMS:
            a = getattr(self, p)
            if cap > n:
                b = np.zeros(cap, np.float64)
                b[:n] = a
                a = b
            bufs[p] = np.ascontiguousarray(a)
        for p in ("active", "frozen"):
            a = getattr(self, p)
            if cap > n:
                b = np.zeros(cap, np.uint8)
                b[:n] = a
                a = b
            bufs[p] = np.ascontiguousarray(a)
        v = _abi.SitesView()
        v.size = n
        v.capacity = cap
        for p in _PARAMS:
            setattr(v, p, bufs[p].ctypes.data_as(C.POINTER(C.c_double)))
        v.active = bufs["active"].ctypes.data_as(C.POINTER(C.c_uint8))
        v.frozen = bufs["frozen"].ctypes.data_as(C.POINTER(C.c_uint8))
        v.generation = self.generation
        return v, bufs

    def _absorb(self, v, bufs):
        n = int(v.size)
        for p in _PARAMS + ("active", "frozen"):
            setattr(self, p, bufs[p][:n].copy())
        self.generation = int(v.generation)


class ImageBuffer:
    """ImageBuffer (types.hpp:67-79): interleaved RGB doubles."""

    def __init__(self, width: int = 0, height: int = 0, data=None):
        self.width = int(width)
        self.height = int(height)
        if data is None:
            self.data = np.zeros(3 * self.width * self.height, np.float64)
        else:
            self.data = np.ascontiguousarray(np.asarray(data, np.float64).reshape(-1))
            if self.data.size != 3 * self.width * self.height:
                raise ValueError("ImageBuffer: data size mismatch")

    def resize(self, w, h):
        if w < 1 or h < 1:
            raise ValueError("ImageBuffer: empty extent")
        self.width, self.height = int(w), int(h)
        self.data = np.zeros(3 * w * h, np.float64)

    def at(self, px, py):
        i = 3 * (py * self.width + px)
        return self.data[i:i + 3]

    def rgb(self) -> np.ndarray:
        return self.data.reshape(self.height, self.width, 3)

    def same_shape(self, o) -> bool:
        return self.width == o.width and self.height == o.height


class CandidateField:
    """CandidateField (types.hpp:84-110)."""
    kEmpty = EMPTY

    def __init__(self):
        self.width = self.height = 0
        self.cell = 1
        self.gw = self.gh = 0
        self.k = 8
        self.ids = np.zeros(0, np.uint32)
        self.synced_generation = (1 << 64) - 1
        self.refresh_count = 0
        self.pass_index = 0

    def resize(self, w, h, k_slots, cell_size=1):
        if w < 1 or h < 1:
            raise ValueError("CandidateField: empty extent")
        if k_slots < 1 or k_slots > 16:
            raise ValueError("CandidateField: k out of range")
        if cell_size < 1:
            raise ValueError("CandidateField: bad cell size")
        self.width, self.height, self.cell = int(w), int(h), int(cell_size)
        self.gw = (w + cell_size - 1) // cell_size
        self.gh = (h + cell_size - 1) // cell_size
        self.k = int(k_slots)
        self.ids = np.full(self.gw * self.gh * self.k, EMPTY, np.uint32)
        self.synced_generation = (1 << 64) - 1

    def slot(self, gx, gy) -> np.ndarray:
        o = self.k * (gy * self.gw + gx)
        return self.ids[o:o + self.k]

    def center_x(self, gx):
        return gx * float(self.cell) + (self.cell - 1) * 0.5

    def center_y(self, gy):
        return gy * float(self.cell) + (self.cell - 1) * 0.5

    def copy(self) -> "CandidateField":
        o = CandidateField()
        o.__dict__.update({k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in self.__dict__.items()})
        return o

    def _view(self):
        self.ids = np.ascontiguousarray(self.ids, dtype=np.uint32)
        v = _abi.FieldView()
        v.width, v.height, v.cell, v.gw, v.gh, v.k = self.width, self.height, self.cell, self.gw, self.gh, self.k
        v.ids = self.ids.ctypes.data_as(C.POINTER(C.c_uint32))
        v.synced_generation = self.synced_generation
        v.refresh_count = self.refresh_count
        v.pass_index = self.pass_index
        return v

    def _absorb(self, v):
        self.synced_generation = int(v.synced_generation)
        self.refresh_count = int(v.refresh_count)
        self.pass_index = int(v.pass_index)


class GradBuffer:
    """GradBuffer (grad.hpp:35-57): n x 11 values of the compensated per-site accumulators."""

    def __init__(self, n: int = 0):
        self.resize(n)

    def resize(self, n):
        self.data = np.zeros((n, kChannels), np.float64)
        self.nonfinite = 0

    def reset(self):
        self.data[:] = 0
        self.nonfinite = 0

    def size(self):
        return self.data.shape[0]

    def grad(self, slot, id):
        return float(self.data[id, slot])

    def removal_delta(self, id):
        return float(self.data[id, kGradSlots])


class AdamState:
    """AdamState (train.hpp:13-21)."""

    def __init__(self, n: int = 0):
        self.m = np.zeros(n * kGradSlots, np.float64)
        self.v = np.zeros(n * kGradSlots, np.float64)
        self.t = 0
        self.skipped = 0

    def sites(self):
        return self.m.shape[0] // kGradSlots

    def resize(self, n):
        m = np.zeros(n * kGradSlots)
        v = np.zeros(n * kGradSlots)
        k = min(n * kGradSlots, self.m.shape[0])
        m[:k], v[:k] = self.m[:k], self.v[:k]
        self.m, self.v = m, v

    def zero_site(self, id):
        if id >= self.sites():
            self.resize(id + 1)
        self.m[id * 10:(id + 1) * 10] = 0
        self.v[id * 10:(id + 1) * 10] = 0

    def _view(self, capacity):
        n = self.sites()
        cap = max(n, capacity, 1)
        m = np.zeros(cap * 10)
        v = np.zeros(cap * 10)
        m[: n * 10], v[: n * 10] = self.m, self.v
        av = _abi.AdamView()
        av.sites, av.capacity = n, cap
        av.m = m.ctypes.data_as(C.POINTER(C.c_double))
        av.v = v.ctypes.data_as(C.POINTER(C.c_double))
        av.t, av.skipped = self.t, self.skipped
        return av, (m, v)

    def _absorb(self, av, bufs):
        n = int(av.sites)
        self.m = bufs[0][: n * 10].copy()
        self.v = bufs[1][: n * 10].copy()
        self.t = int(av.t)
        self.skipped = int(av.skipped)


@dataclass
class SiteStats:
    mass: float = 0
    energy: float = 0
    sx: float = 0
    sy: float = 0
    sxx: float = 0
    sxy: float = 0
    syy: float = 0
    removal: float = 0


class StatsResult:
    """StatsResult (budget.hpp:22-25): `data` is n x 8 (mass, energy, sx, sy, sxx, sxy, syy, removal)."""

    def __init__(self, n=0):
        self.data = np.zeros((n, 8), np.float64)
        self.valid_pixels = 0

    @property
    def site(self):
        return [SiteStats(*map(float, r)) for r in self.data]


@dataclass
class LearningRates:
    pos: float = 0.5
    color: float = 0.05
    log_tau: float = 0.05
    radius: float = 0.25
    dir: float = 0.025
    aniso: float = 0.025


@dataclass
class TrainConfig:
    """TrainConfig (types.hpp:121-167) with the reference defaults."""
    iters: int = 4000
    n_sites: int = 0
    target_bpp: float = 0.0
    seed: int = 1
    k: int = 8
    inject: int = 4
    lambda_init: float = 0.3
    lr: LearningRates = field(default_factory=LearningRates)
    beta1: float = 0.9
    beta2: float = 0.999
    adam_eps: float = 1e-8
    refresh_every: int = 1
    refresh_passes: int = 1
    final_passes: int = 16
    tau_diffusion_lambda: float = 0.0
    densify_every: int = 20
    densify_start: int = 20
    densify_end: int = 3000
    densify_pct: float = 0.01
    alpha: float = 0.7
    stats_eps: float = 1e-8
    prune_every: int = 40
    prune_start: int = 100
    prune_end: int = 3000
    prune_pct: float = 0.033
    prune_during_densify: bool = True
    budget_scale_cap: float = 0.95
    max_sites: int = 0
    init_log_tau: float = 7.5
    init_radius: float = 0.0
    init_aniso: float = 0.0
    log_tau_min: float = 2.0
    log_tau_max: float = 20.0
    radius_min: float = 1.0
    radius_max: float = 512.0
    aniso_min: float = -2.0
    aniso_max: float = 2.0
    clamp_color: bool = True
    fp64: bool = True
    threads: int = 1

    def to_c(self) -> _abi.TrainConfigC:
        c = _abi.TrainConfigC()
        for f in dataclasses.fields(self):
            if f.name == "lr":
                for lf in dataclasses.fields(LearningRates):
                    setattr(c, "lr_" + lf.name, getattr(self.lr, lf.name))
            else:
                v = getattr(self, f.name)
                setattr(c, f.name, int(v) if isinstance(v, bool) else v)
        return c

    def copy(self) -> "TrainConfig":
        return dataclasses.replace(self, lr=dataclasses.replace(self.lr))


def run_opts(cfg: TrainConfig) -> RunOpts:
    return RunOpts(cfg.fp64, cfg.threads)


@dataclass
class HistoryRow:
    """HistoryRow (train.hpp:46-52)."""
    iter: int = 0
    loss: float = 0.0
    psnr: float = 0.0
    active_sites: int = 0
    ms: float = 0.0


def history_line(r: HistoryRow) -> str:
    """history_line (train.cpp:317-321): %d,%.17g,%.17g,%d."""
    return "%d,%.17g,%.17g,%d" % (r.iter, r.loss, r.psnr, r.active_sites)


@dataclass
class FitResult:
    """FitResult (train.hpp:54-59)."""
    sites: SiteStore
    field: CandidateField
    history: List[HistoryRow]
    schedule_scale: float = 0.0
    timing: Optional[dict] = None


def normalization_scale(width: int, height: int) -> float:
    """normalization_scale (types.hpp:178-181)."""
    if width < 1 or height < 1:
        raise ValueError("normalization_scale: empty extent")
    return 1.0 / float(max(width, height))


def psnr_from_loss(loss: float) -> float:
    """psnr_from_loss (quality.cpp:68-73)."""
    import math
    m = loss / 3.0
    if m <= 0:
        return 99.0
    v = 10.0 * math.log10(1.0 / m)
    return 99.0 if v > 99.0 else v
