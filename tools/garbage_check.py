"""Fits after the device memory was filled with garbage and released (uninitialised-read hunting): each run
first fills ~GB of device memory with random bytes through torch, frees it, then runs the golden fit.
    python tools/garbage_check.py tests/golden/fit_config2_s7.npz 6"""
import ast
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_21984_b200 as sad  # noqa: E402
from paper_2604_21984_b200.synth import synthetic_image  # noqa: E402

path, reps = sys.argv[1], int(sys.argv[2])
d = np.load(path)
w, h, seed = int(d["width"]), int(d["height"]), int(d["image_seed"])
cfg = sad.TrainConfig(**ast.literal_eval(str(d["config"])))
img = sad.ImageBuffer(w, h, synthetic_image(w, h, seed))
P = ("x", "y", "log_tau", "radius", "col_r", "col_g", "col_b", "dir_x", "dir_y", "aniso", "active", "frozen")
for i in range(reps):
    g = torch.randint(0, 256, (int(os.environ.get("GB", 8)) << 30,), dtype=torch.uint8, device="cuda")
    del g
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    G = sad.gpu_backend(0)
    res = G.fit(img, cfg)
    loss = np.array([r.loss for r in res.history], np.float64)
    first = np.flatnonzero(loss.view(np.uint64) != d["loss"].view(np.uint64))
    bad = [p for p in P if hashlib.sha256(np.ascontiguousarray(getattr(res.sites, p)).tobytes()).hexdigest() != str(d["sha_" + p])]
    field_ok = hashlib.sha256(res.field.ids.tobytes()).hexdigest() == str(d["field_sha"])
    print(f"run {i}: history {'ok' if first.size == 0 else 'DIFF from ' + str(first[0] + 1)} sites {bad or 'ok'} "
          f"field {'ok' if field_ok else 'DIFF'}", flush=True)
