"""fp64 config-2 fit against its committed reference golden: first differing history row, site digests.
    python tools/fp64_golden_check.py [tests/golden/fit_config2_fp64_s1.npz]"""
import ast
import hashlib
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2604_21984_b200 as sad  # noqa: E402
from paper_2604_21984_b200.synth import synthetic_image  # noqa: E402

path = sys.argv[1] if len(sys.argv) > 1 else "tests/golden/fit_config2_fp64_s1.npz"
d = np.load(path)
w, h, seed = int(d["width"]), int(d["height"]), int(d["image_seed"])
cfg = sad.TrainConfig(**ast.literal_eval(str(d["config"])))
img = sad.ImageBuffer(w, h, synthetic_image(w, h, seed))
G = sad.gpu_backend(0)
t0 = time.perf_counter()
res = G.fit(img, cfg)
sec = time.perf_counter() - t0
loss = np.array([r.loss for r in res.history], np.float64)
active = np.array([r.active_sites for r in res.history], np.int64)
bad = np.flatnonzero((loss.view(np.uint64) != d["loss"].view(np.uint64)) | (active != d["active"]))
print(f"{os.path.basename(path)}: {len(loss)} rows, first differing row {bad[0] + 1 if bad.size else None}, "
      f"fit {sec:.2f} s")
for p in ("x", "y", "log_tau", "radius", "col_r", "col_g", "col_b", "dir_x", "dir_y", "aniso", "active", "frozen"):
    ok = hashlib.sha256(np.ascontiguousarray(getattr(res.sites, p)).tobytes()).hexdigest() == str(d["sha_" + p])
    print(f"  {p}: {'identical' if ok else 'DIFFERS'}")
print("  field:", "identical" if hashlib.sha256(res.field.ids.tobytes()).hexdigest() == str(d["field_sha"]) else "DIFFERS")
