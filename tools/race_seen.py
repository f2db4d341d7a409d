"""For fits whose final site arrays differ between runs: are the differing sites held by any candidate list?
    SAD_STOP_AT=3990 python tools/race_seen.py REPS"""
import ast
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
first = G.fit(img, cfg)
ids = first.field.ids
seen = np.zeros(first.sites.size(), bool)
seen[ids[ids < first.sites.size()]] = True
print("site 71 in the final map:", bool(seen[71]), "count", int((ids == 71).sum()), flush=True)
for i in range(reps):
    res = G.fit(img, cfg)
    for p in ("x", "y", "log_tau", "radius", "col_r", "col_g", "col_b", "dir_x", "dir_y", "aniso"):
        diff = np.flatnonzero(getattr(res.sites, p) != getattr(first.sites, p))
        if diff.size:
            print(f"run {i}: {p} differs at {diff[:6]}, held by the map: {seen[diff].tolist()[:6]}", flush=True)
