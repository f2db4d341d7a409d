"""Per-phase clock64 totals of k_backward from an SAD_EXPERIMENT=3 build (exp/libsad_exp3.so).
   python tools/phase_clk.py exp/libsad_exp3.so"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_21984_b200 as sad  # noqa: E402
from paper_2604_21984_b200 import api  # noqa: E402
from paper_2604_21984_b200.synth import synthetic_image  # noqa: E402

api.LIB_PATH = os.path.abspath(sys.argv[1])
G = sad.gpu_backend(0)
cfg = sad.TrainConfig(iters=int(os.environ.get('ITERS', 200)), target_bpp=2.0, fp64=False)
run = C.c_void_p()
cc = cfg.to_c()
G._call("fit_create", C.c_int(768), C.c_int(512), C.byref(cc), C.byref(run))
img = synthetic_image(768, 512, 1)
G._call("fit_set_target", run, img.ctypes.data_as(C.POINTER(C.c_double)))
G._call("fit_run_init", run)
buf = (C.c_ulonglong * 16)()
G.lib.sad_exp_phase(buf, 1)
out = C.c_double()
G._call("fit_bench", run, C.c_int(1), C.c_int(20), C.byref(out))
G.lib.sad_exp_phase(buf, 0)
names = ["phase1(fwd+bwd math)", "hash insert", "compact+slot claim", "count+scan", "scatter", "chunk scan+fill",
         "dd sums half A (+store)", "dd sums half B (+store)", "merge+records"]
blocks = 21 * 3072  # 1 warm-up + 20 timed launches
tot = sum(buf[i] for i in range(9))
for i, nm in enumerate(names):
    print(f"{nm:24s} {buf[i] / blocks:10.0f} cycles/block  {100.0 * buf[i] / tot:5.1f}%")
print(f"us/launch (event) {out.value * 1e3:.1f}  CAS-fallback site records: {buf[15] / 21:.0f} per launch")
print(f"entries kept {buf[13] / 21:.0f} per launch, with w == 0: {100.0 * buf[14] / max(buf[13], 1):.1f}%")
