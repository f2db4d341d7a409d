"""Per-phase CUDA-event totals of one resident fit (profiling mode: no graphs, an event pair per phase),
printed by the library on stderr: propagate (warm + event refresh passes), fwd+bwd, Adam, events (stats,
selection, compaction, seeding), advance.
    W=768 H=512 ITERS=4000 python tools/phase_fit.py"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_21984_b200 as sad  # noqa: E402
from paper_2604_21984_b200.synth import synthetic_image  # noqa: E402

W, H = int(os.environ.get("W", 768)), int(os.environ.get("H", 512))
cfg = sad.TrainConfig(iters=int(os.environ.get("ITERS", 4000)), target_bpp=2.0, fp64=os.environ.get("FP64") == "1")
G = sad.gpu_backend(0)
run = C.c_void_p()
cc = cfg.to_c()
G._call("fit_create", C.c_int(W), C.c_int(H), C.byref(cc), C.byref(run))
img = synthetic_image(W, H, 1)
G._call("fit_set_target", run, img.ctypes.data_as(C.POINTER(C.c_double)))
for prof in (0, 1):
    G._call("fit_set_profiling", run, C.c_int(prof))
    G._call("fit_run_init", run)
    tot, ph = C.c_double(), (C.c_double * 4)()
    G._call("fit_timing", run, C.byref(tot), ph)
    print(f"{W}x{H} iters {cfg.iters} profiling={prof}: total {tot.value:.1f} ms, phases {[round(x, 1) for x in ph]}",
          flush=True)
