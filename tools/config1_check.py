"""Config 1: 256x256 synthetic image, n_sites 4096, 200 iterations, budget off, fp32 and
fp64.  The GPU fit vs the compiled reference at 1 thread and at all host threads: history identity and
wall times.   python tools/config1_check.py"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_21984_b200 as sad  # noqa: E402
from oracle.bindings import ref_backend  # noqa: E402
from paper_2604_21984_b200.synth import synthetic_image  # noqa: E402

G = sad.gpu_backend(0)
img = sad.ImageBuffer(256, 256, synthetic_image(256, 256, 1))
allt = os.cpu_count() or 1
for fp64 in (False, True):
    cfg = sad.TrainConfig(iters=200, n_sites=4096, fp64=fp64, seed=1)
    G.fit(img, cfg)
    t0 = time.perf_counter()
    a = G.fit(img, cfg)
    tg = time.perf_counter() - t0
    line = [f"fp{'64' if fp64 else '32'}: gpu {tg * 1e3:.1f} ms ({200 / tg:.0f} iters/s)"]
    for th in (1, allt):
        R = ref_backend(threads=th)
        c = sad.TrainConfig(iters=200, n_sites=4096, fp64=fp64, seed=1)
        c.threads = th
        t0 = time.perf_counter()
        b = R.fit(img, c)
        tr = time.perf_counter() - t0
        same = [sad.history_line(r) for r in a.history] == [sad.history_line(r) for r in b.history]
        same = same and np.array_equal(a.sites.x, b.sites.x) and np.array_equal(a.field.ids, b.field.ids)
        line.append(f"reference {th} thread(s) {tr:.2f} s ({200 / tr:.1f} iters/s), identical {same}")
    print("; ".join(line), f"; final PSNR {a.history[-1].psnr:.4f}", flush=True)
