"""Run the same fit many times in one process and count runs whose final state differs from the first's
(nondeterminism hunting).   ITERS=400 SEED=7 REPS=60 python tools/race_stress.py"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2604_21984_b200 as sad  # noqa: E402
from paper_2604_21984_b200.synth import synthetic_image  # noqa: E402

iters, seed, reps = int(os.environ.get("ITERS", 400)), int(os.environ.get("SEED", 7)), int(os.environ.get("REPS", 60))
W, H = 768, 512
img = sad.ImageBuffer(W, H, synthetic_image(W, H, seed))
cfg = sad.TrainConfig(iters=iters, target_bpp=2.0, fp64=os.environ.get("FP64") == "1")
G = sad.gpu_backend(0)
P = ("x", "y", "log_tau", "radius", "col_r", "col_g", "col_b", "dir_x", "dir_y", "aniso", "active")


def digest(res):
    out = {p: hashlib.sha256(np.ascontiguousarray(getattr(res.sites, p)).tobytes()).hexdigest()[:12] for p in P}
    out["field"] = hashlib.sha256(res.field.ids.tobytes()).hexdigest()[:12]
    out["hist"] = hashlib.sha256(np.array([r.loss for r in res.history]).tobytes()).hexdigest()[:12]
    return out


ref = digest(G.fit(img, cfg))
bad = 0
for i in range(reps):
    d = digest(G.fit(img, cfg))
    diff = [k for k in d if d[k] != ref[k]]
    if diff:
        bad += 1
        print(f"run {i}: differs in {diff}", flush=True)
print(f"{reps} runs, {bad} differ from the first (iters {iters}, seed {seed})")
