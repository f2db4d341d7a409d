"""Python restatements of the reference test fixtures (seeded generators), so parity tests build
the same inputs the reference's own doctest suites use."""
from __future__ import annotations

import math

import numpy as np

from paper_2604_21984_b200 import ImageBuffer, Site, SiteStore
from paper_2604_21984_b200.synth import Rng, synthetic_image


def random_sites(w, h, n, seed) -> SiteStore:
    """test_candidates.cpp:15-33: collision-free cells plus subpixel offsets."""
    st = SiteStore(0)
    rng = Rng(seed, 0xC0FFEE, 0)
    cells = list(range(w * h))
    for i in range(n):
        j = i + rng.next_below(len(cells) - i)
        cells[i], cells[j] = cells[j], cells[i]
        x = (cells[i] % w) + rng.next_unit() * 0.5 + 0.25
        y = (cells[i] // w) + rng.next_unit() * 0.5 + 0.25
        st.append(Site(x=min(x, w - 1.0), y=min(y, h - 1.0), log_tau=7.5, radius=math.sqrt(w * h / n)))
    return st


def random_model(w, h, n, seed) -> SiteStore:
    """test_grad.cpp:16-33 / test_render.cpp:16-33 / test_budget.cpp:18-35."""
    st = SiteStore(0)
    rng = Rng(seed, 0xBEEF, 1)
    for _ in range(n):
        x = rng.next_unit() * (w - 1)
        y = rng.next_unit() * (h - 1)
        lt = 6.0 + rng.next_unit() * 3.0
        r = 1.0 + rng.next_unit() * 8.0
        col = tuple(rng.next_unit() for _ in range(3))
        th = rng.next_unit() * 6.283185307179586
        a = (rng.next_unit() - 0.5) * 2.0
        st.append(Site(x=x, y=y, log_tau=lt, radius=r, color=col, dir=(math.cos(th), math.sin(th)), aniso=a))
    return st


def random_target(w, h, seed) -> ImageBuffer:
    """test_grad.cpp:35-41: every value from seeded_stream(seed, 0x515, 2)."""
    rng = Rng(seed, 0x515, 2)
    return ImageBuffer(w, h, [rng.next_unit() for _ in range(3 * w * h)])


def constant_image(w, h, r, g, b) -> ImageBuffer:
    img = ImageBuffer(w, h)
    img.data.reshape(-1, 3)[:] = (r, g, b)
    return img


def ramp_image(w, h) -> ImageBuffer:
    """A smooth two-axis colour ramp."""
    y, x = np.mgrid[0:h, 0:w].astype(np.float64)
    d = np.stack([x / max(w - 1, 1), y / max(h - 1, 1), 0.5 * (x / max(w - 1, 1) + y / max(h - 1, 1))], -1)
    return ImageBuffer(w, h, d.reshape(-1))


def synth_target(w, h, seed=1) -> ImageBuffer:
    return ImageBuffer(w, h, synthetic_image(w, h, seed))
