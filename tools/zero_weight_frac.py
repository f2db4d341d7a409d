"""Fraction of kept candidates whose fp32 softmax weight underflows to exactly 0 (logit - best < -103.97,
glibc expf's underflow bound) on a fitted field: the work a zero-weight shortcut in render / fwd+bwd would
skip.   python tools/zero_weight_frac.py [--width 768 --height 512 --iters 4000]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2604_21984_b200 as sad  # noqa: E402
from paper_2604_21984_b200.synth import synthetic_image  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--width", type=int, default=768)
ap.add_argument("--height", type=int, default=512)
ap.add_argument("--iters", type=int, default=4000)
ap.add_argument("--n-sites", type=int, default=0)
a = ap.parse_args()
G = sad.gpu_backend(0)
W, H = a.width, a.height
cfg = sad.TrainConfig(iters=a.iters, target_bpp=0.0 if a.n_sites else 2.0, n_sites=a.n_sites, fp64=False)
res = G.fit(sad.ImageBuffer(W, H, synthetic_image(W, H, 1)), cfg)
yy, xx = np.mgrid[0:H, 0:W]
pix = np.stack([xx.ravel(), yy.ravel()], 1).astype(np.int32)
tot = zero = 0
for i in range(0, pix.shape[0], 500_000):
    ids, w, n = G.pixel_weights_batch(res.sites, res.field, pix[i:i + 500_000])
    mask = np.arange(16)[None, :] < n[:, None]
    tot += int(mask.sum())
    zero += int((mask & (w < 7.0e-46)).sum())
print(f"{W}x{H}, {a.iters} iterations: {zero} of {tot} kept candidates ({100.0 * zero / tot:.1f}%) have an fp32 weight of 0")
