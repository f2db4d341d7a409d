"""Repeat the seed-7 config-2 fit; for runs whose radius differs from the golden, print the differing sites.
    python tools/race_detail.py REPS"""
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
good = None
bads = []
for i in range(reps):
    res = G.fit(img, cfg)
    r = res.sites.radius.copy()
    ok = hashlib.sha256(np.ascontiguousarray(r).tobytes()).hexdigest() == str(d["sha_radius"])
    if ok and good is None:
        good = res
    if not ok:
        bads.append(res)
        print(f"run {i}: radius differs", flush=True)
    if good is not None and bads:
        for b in bads:
            idx = np.flatnonzero(b.sites.radius != good.sites.radius)
            print("  sites", idx[:10], "good", good.sites.radius[idx[:5]], "bad", b.sites.radius[idx[:5]],
                  "active", good.sites.active[idx[:5]], b.sites.active[idx[:5]], "frozen", good.sites.frozen[idx[:5]],
                  flush=True)
            for p in ("x", "y", "log_tau", "col_r", "aniso", "dir_x"):
                if not np.array_equal(getattr(b.sites, p), getattr(good.sites, p)):
                    print("  also differs:", p, flush=True)
        bads = []
