"""Nondeterminism check of fits stopped early (SAD_STOP_AT): final site arrays compared across runs.
    SAD_STOP_AT=3990 python tools/race_stop.py REPS"""
import ast
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2604_21984_b200 as sad  # noqa: E402
from paper_2604_21984_b200.synth import synthetic_image  # noqa: E402

reps = int(sys.argv[1])
d = np.load("tests/golden/fit_config2_s7.npz")
w, h, seed = int(d["width"]), int(d["height"]), int(d["image_seed"])
cfg = sad.TrainConfig(**ast.literal_eval(str(d["config"])))
img = sad.ImageBuffer(w, h, synthetic_image(w, h, seed))
G = sad.gpu_backend(0)
P = ("x", "y", "log_tau", "radius", "col_r", "col_g", "col_b", "dir_x", "dir_y", "aniso")
counts = {}
first = None
for i in range(reps):
    res = G.fit(img, cfg)
    dg = tuple(hashlib.sha256(np.ascontiguousarray(getattr(res.sites, p)).tobytes()).hexdigest()[:10] for p in P)
    counts[dg] = counts.get(dg, 0) + 1
    if first is None:
        first = res
    elif dg != tuple(hashlib.sha256(np.ascontiguousarray(getattr(first.sites, p)).tobytes()).hexdigest()[:10] for p in P):
        for p in P:
            a, b = getattr(first.sites, p), getattr(res.sites, p)
            idx = np.flatnonzero(a != b)
            if idx.size:
                print(f"run {i}: {p} differs at {idx[:8]} ({a[idx[0]]!r} vs {b[idx[0]]!r})", flush=True)
print(f"stop_at {os.environ.get('SAD_STOP_AT')}: {len(counts)} distinct outcomes {sorted(counts.values(), reverse=True)}")
