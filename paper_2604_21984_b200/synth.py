"""Seeded synthetic inputs (not part of the hot path): the reference's counter-seeded xorshift
streams (rng.hpp:12-45) in Python/numpy, and the procedural RGB test image used by the bench and
the parity tests (smooth trig background, 12 hard-edged discs, +-0.01 noise from
seeded_stream(seed, 0x5157, .), quantised to k/255 like an 8-bit PNG).
"""
from __future__ import annotations

import math

import numpy as np

M32 = 0xFFFFFFFF


def mix32(h: int) -> int:
    h &= M32
    h ^= h >> 16
    h = (h * 0x7FEB352D) & M32
    h ^= h >> 15
    h = (h * 0x846CA68B) & M32
    h ^= h >> 16
    return h


def seeded_state(seed: int, a: int, b: int) -> int:
    h = mix32((seed & M32) ^ 0x9E3779B9)
    h ^= mix32(((seed >> 32) + 0x85EBCA6B) & M32)
    h = mix32((h + mix32((a ^ 0x27D4EB2F) & M32)) & M32)
    h = mix32(h ^ mix32((b + 0x165667B1) & M32))
    return h if h else 0x6B33A1C9


class Rng:
    """RngState (rng.hpp:9-26)."""

    def __init__(self, seed: int, a: int, b: int):
        self.s = seeded_state(seed, a, b)

    def next(self) -> int:
        x = self.s
        x ^= (x << 13) & M32
        x ^= x >> 17
        x ^= (x << 5) & M32
        self.s = x
        return x

    def next_unit(self) -> float:
        return (self.next() >> 8) * (1.0 / 16777216.0)

    def next_below(self, n: int) -> int:
        return self.next() % n if n else 0


def _xs_vec(s: np.ndarray) -> np.ndarray:
    s = s ^ (s << np.uint32(13))
    s = s ^ (s >> np.uint32(17))
    s = s ^ (s << np.uint32(5))
    return s


def synthetic_image(width: int, height: int, seed: int = 1, quantize: bool = True) -> np.ndarray:
    """Procedural RGB image in [0,1], interleaved [py][px][c] doubles (ImageBuffer layout)."""
    rng = Rng(seed, 0x5157, 0)
    y, x = np.mgrid[0:height, 0:width].astype(np.float64)
    u, v = x / max(width - 1, 1), y / max(height - 1, 1)
    f = [1.0 + 3.0 * rng.next_unit() for _ in range(6)]
    ph = [2.0 * math.pi * rng.next_unit() for _ in range(6)]
    img = np.empty((height, width, 3), np.float64)
    for c in range(3):
        img[..., c] = 0.5 + 0.22 * np.sin(2 * math.pi * f[2 * c] * u + ph[2 * c]) * np.cos(
            2 * math.pi * f[2 * c + 1] * v + ph[2 * c + 1]) + 0.12 * (u - 0.5) * (1 if c == 1 else -1)
    rmax = 0.18 * min(width, height)
    for _ in range(12):
        cx, cy = rng.next_unit() * width, rng.next_unit() * height
        r = (0.25 + 0.75 * rng.next_unit()) * rmax
        col = [rng.next_unit() for _ in range(3)]
        m = (x - cx) ** 2 + (y - cy) ** 2 <= r * r
        img[m] = col
    # +-0.01 uniform noise: one xorshift stream per row, 3 draws per pixel in raster order
    s = np.array([seeded_state(seed, 0x5157, 1 + r) for r in range(height)], np.uint32)
    noise = np.empty((height, width * 3), np.float64)
    for j in range(width * 3):
        s = _xs_vec(s)
        noise[:, j] = (s >> np.uint32(8)).astype(np.float64) * (1.0 / 16777216.0)
    img += (noise.reshape(height, width, 3) - 0.5) * 0.02
    img = np.clip(img, 0.0, 1.0)
    if quantize:
        img = np.round(img * 255.0) / 255.0
    return np.ascontiguousarray(img.reshape(-1))
