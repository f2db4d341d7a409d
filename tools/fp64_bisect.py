"""First event iteration at which the fp64 config-2 GPU fit's sites differ from the reference's.
    python tools/fp64_bisect.py T1 T2 ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2604_21984_b200 as sad  # noqa: E402
from oracle.bindings import ref_backend  # noqa: E402
from paper_2604_21984_b200.synth import synthetic_image  # noqa: E402

img = sad.ImageBuffer(768, 512, synthetic_image(768, 512, 1))
G = sad.gpu_backend(0)
R = ref_backend(threads=os.cpu_count() or 1)
P = ("x", "y", "log_tau", "radius", "col_r", "col_g", "col_b", "dir_x", "dir_y", "aniso", "active")
for T in (int(v) for v in sys.argv[1:]):
    out = []
    for B, env in ((G, "SAD_STOP_AT"), (R, "SAD_REF_STOP_AT")):
        os.environ[env] = str(T)
        cfg = sad.TrainConfig(iters=4000, target_bpp=2.0, fp64=True, seed=1)
        cfg.threads = os.cpu_count() or 1
        out.append(B.fit(img, cfg))
        del os.environ[env]
    a, b = out
    diff = sorted(set(np.concatenate([np.flatnonzero(getattr(a.sites, p) != getattr(b.sites, p)) for p in P])))
    print(T, "sites", a.sites.size(), b.sites.size(), "differing", diff[:20], flush=True)
    if diff:
        np.savez_compressed(f"gpurun_out/bisect_{T}.npz", **{f"g_{p}": getattr(a.sites, p) for p in P},
                            **{f"r_{p}": getattr(b.sites, p) for p in P}, g_ids=a.field.ids, r_ids=b.field.ids)
