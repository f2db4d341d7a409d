"""Times complete fits: device-resident (fit_run_init on a reused run) and end-to-end (Backend.fit).
   python tools/fit_time.py [--width 768 --height 512 --bpp 2 --iters 4000 --reps 3]"""
import argparse
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_21984_b200 as sad  # noqa: E402
from paper_2604_21984_b200.synth import synthetic_image  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--width", type=int, default=768)
p.add_argument("--height", type=int, default=512)
p.add_argument("--bpp", type=float, default=2.0)
p.add_argument("--iters", type=int, default=4000)
p.add_argument("--reps", type=int, default=3)
p.add_argument("--lib", default=None, help="alternative libsad_b200.so (A/B)")
p.add_argument("--no-e2e", action="store_true")
a = p.parse_args()
if a.lib:
    from paper_2604_21984_b200 import api
    api.LIB_PATH = os.path.abspath(a.lib)
G = sad.gpu_backend(0)
cfg = sad.TrainConfig(iters=a.iters, target_bpp=a.bpp, fp64=False)
img = synthetic_image(a.width, a.height, 1)
run = C.c_void_p()
cc = cfg.to_c()
t0 = time.perf_counter()
G._call("fit_create", C.c_int(a.width), C.c_int(a.height), C.byref(cc), C.byref(run))
t1 = time.perf_counter()
G._call("fit_set_target", run, img.ctypes.data_as(C.POINTER(C.c_double)))
if os.environ.get("SAD_PROFILE"):
    G._call("fit_set_profiling", run, C.c_int(1))
print(f"fit_create {1e3 * (t1 - t0):.1f} ms")
for i in range(a.reps):
    t0 = time.perf_counter()
    G._call("fit_run_init", run)
    t1 = time.perf_counter()
    tot, ph = C.c_double(), (C.c_double * 4)()
    G._call("fit_timing", run, C.byref(tot), ph)
    print(f"resident fit {i}: wall {1e3 * (t1 - t0):.1f} ms, device {tot.value:.1f} ms, phases "
          f"propagate {ph[0]:.1f} fwd_bwd {ph[1]:.1f} adam+adv {ph[2]:.1f} events {ph[3]:.1f} ms")
G.lib.sad_fit_destroy(run)
for i in range(0 if a.no_e2e else a.reps):
    t0 = time.perf_counter()
    r = G.fit(sad.ImageBuffer(a.width, a.height, img), cfg)
    print(f"e2e fit {i}: {1e3 * (time.perf_counter() - t0):.1f} ms  psnr_last {r.history[-1].psnr:.3f}")
