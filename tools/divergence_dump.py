"""Divergence hunting: fit a synthetic image and stop after iteration t (SAD_STOP_AT on the GPU,
SAD_REF_STOP_AT on the reference), then save the sites, the candidate map and the history.
    python tools/divergence_dump.py gpu|ref T out.npz [--fp64] [--width 768 --height 512 --seed 1]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2604_21984_b200 as sad  # noqa: E402
from paper_2604_21984_b200.synth import synthetic_image  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("which")
ap.add_argument("t", type=int)
ap.add_argument("out")
ap.add_argument("--fp64", action="store_true")
ap.add_argument("--width", type=int, default=768)
ap.add_argument("--height", type=int, default=512)
ap.add_argument("--seed", type=int, default=1)
a = ap.parse_args()
img = sad.ImageBuffer(a.width, a.height, synthetic_image(a.width, a.height, a.seed))
cfg = sad.TrainConfig(iters=4000, target_bpp=2.0, fp64=a.fp64, seed=1)
if a.which == "gpu":
    os.environ["SAD_STOP_AT"] = str(a.t)
    B = sad.gpu_backend(0)
else:
    from oracle.bindings import ref_backend
    os.environ["SAD_REF_STOP_AT"] = str(a.t)
    cfg.threads = os.cpu_count() or 1
    B = ref_backend(threads=cfg.threads)
res = B.fit(img, cfg)
d = {p: getattr(res.sites, p) for p in ("x", "y", "log_tau", "radius", "col_r", "col_g", "col_b", "dir_x", "dir_y",
                                         "aniso", "active", "frozen")}
d["ids"] = res.field.ids
d["loss"] = np.array([r.loss for r in res.history])
d["active_hist"] = np.array([r.active_sites for r in res.history])
np.savez_compressed(a.out, **d)
print(a.which, a.t, len(res.history), res.sites.size())
