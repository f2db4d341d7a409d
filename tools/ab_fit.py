"""A/B: config-2 fit with an alternative library: digest of history/sites/map + resident fit times.
   python tools/ab_fit.py exp/libsad_TAG.so [iters]"""
import ctypes as C, hashlib, os, sys
sys.path.insert(0, "/root/repo")
from paper_2604_21984_b200 import api
api.LIB_PATH = os.path.abspath(sys.argv[1])
import paper_2604_21984_b200 as sad
from paper_2604_21984_b200.synth import synthetic_image
from paper_2604_21984_b200.types import _PARAMS
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 4000
W, H = int(os.environ.get("W", 768)), int(os.environ.get("H", 512))
G = sad.gpu_backend(0)
cfg = sad.TrainConfig(iters=iters, target_bpp=2.0, fp64=os.environ.get("FP64") == "1")
img = synthetic_image(W, H, 1)
r = G.fit(sad.ImageBuffer(W, H, img), cfg)
h = hashlib.sha256()
for row in r.history:
    h.update(repr((row.iter, row.loss, row.psnr, row.active_sites)).encode())
for p in _PARAMS:
    h.update(getattr(r.sites, p).tobytes())
h.update(r.field.ids.tobytes())
run = C.c_void_p(); cc = cfg.to_c()
G._call("fit_create", C.c_int(W), C.c_int(H), C.byref(cc), C.byref(run))
G._call("fit_set_target", run, img.ctypes.data_as(C.POINTER(C.c_double)))
ts = []
for i in range(4):
    G._call("fit_run_init", run)
    tot, ph = C.c_double(), (C.c_double * 4)()
    G._call("fit_timing", run, C.byref(tot), ph)
    ts.append(tot.value)
print(f"{os.path.basename(sys.argv[1])}: digest {h.hexdigest()[:16]} psnr {r.history[-1].psnr:.6f} fit ms {' '.join(f'{t:.1f}' for t in ts)}")
