"""Kernel micro-benchmark driver (for ncu captures): fits a synthetic image for a few hundred
iterations, then launches one kernel `--reps` times on the fitted device-resident state.

  python tools/kbench.py --kernel fwd_bwd --reps 20 [--width 768 --height 512 --iters 200]
"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2604_21984_b200 as sad  # noqa: E402
from paper_2604_21984_b200 import api  # noqa: E402
from paper_2604_21984_b200.synth import synthetic_image  # noqa: E402

KERNELS = {"propagate_warm": 0, "fwd_bwd": 1, "render": 2, "propagate_flood": 3, "adam": 4, "stats": 5,
           "memsets": 6, "refresh_full": 7, "box_step": 8,
           "adam_active": 9, "advance": 10}

p = argparse.ArgumentParser()
p.add_argument("--kernel", default="fwd_bwd", help="one of %s, or a comma-separated list (one fit, several kernels)" % list(KERNELS))
p.add_argument("--reps", type=int, default=20)
p.add_argument("--width", type=int, default=768)
p.add_argument("--height", type=int, default=512)
p.add_argument("--iters", type=int, default=200)
p.add_argument("--bpp", type=float, default=2.0)
p.add_argument("--n-sites", type=int, default=0)
p.add_argument("--lib", default=None, help="alternative libsad_b200.so (ablation builds)")
a = p.parse_args()

if a.lib:
    api.LIB_PATH = a.lib
G = sad.gpu_backend(0)
cfg = sad.TrainConfig(iters=a.iters, target_bpp=a.bpp if not a.n_sites else 0.0, n_sites=a.n_sites, fp64=False)
run = C.c_void_p()
cc = cfg.to_c()
G._call("fit_create", C.c_int(a.width), C.c_int(a.height), C.byref(cc), C.byref(run))
img = synthetic_image(a.width, a.height, 1)
G._call("fit_set_target", run, img.ctypes.data_as(C.POINTER(C.c_double)))
G._call("fit_run_init", run)
out = C.c_double()
for kn in a.kernel.split(","):
    G._call("fit_bench", run, C.c_int(KERNELS[kn]), C.c_int(a.reps), C.byref(out))
    print(f"{kn}: {out.value * 1e3:.2f} us/launch ({a.width}x{a.height})")
G.lib.sad_fit_destroy(run)
