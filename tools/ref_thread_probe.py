"""Is the reference's fp64 config-2 fit thread-count invariant?  Fits to iteration T with two worker counts
and compares the site arrays.   python tools/ref_thread_probe.py T threads_a threads_b"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2604_21984_b200 as sad  # noqa: E402
from oracle.bindings import ref_backend  # noqa: E402
from paper_2604_21984_b200.synth import synthetic_image  # noqa: E402

T, ta, tb = (int(v) for v in sys.argv[1:4])
img = sad.ImageBuffer(768, 512, synthetic_image(768, 512, 1))
os.environ["SAD_REF_STOP_AT"] = str(T)
res = []
for th in (ta, tb):
    cfg = sad.TrainConfig(iters=4000, target_bpp=2.0, fp64=True, seed=1)
    cfg.threads = th
    res.append(ref_backend(threads=th).fit(img, cfg))
a, b = res
for p in ("x", "y", "log_tau", "radius", "dir_x", "aniso", "active"):
    d = np.flatnonzero(getattr(a.sites, p) != getattr(b.sites, p))
    print(f"threads {ta} vs {tb}: {p} differs at", d[:12])
print("history identical", [sad.history_line(r) for r in a.history] == [sad.history_line(r) for r in b.history])
