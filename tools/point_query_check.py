"""Resident batched point queries (sad_fit_point_query) vs the per-call pixel_weights API, plus timing.
   python tools/point_query_check.py [W] [nq]"""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_21984_b200 as sad  # noqa: E402
from paper_2604_21984_b200.synth import synthetic_image  # noqa: E402

W = H = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
G = sad.gpu_backend(0)
cfg = sad.TrainConfig(iters=50, n_sites=max(6000, W * H // 42), fp64=False)
run = C.c_void_p()
cc = cfg.to_c()
G._call("fit_create", C.c_int(W), C.c_int(H), C.byref(cc), C.byref(run))
img = synthetic_image(W, H, 3)
G._call("fit_set_target", run, img.ctypes.data_as(C.POINTER(C.c_double)))
G._call("fit_run_init", run)
rng = np.random.default_rng(0)
xy = np.stack([rng.integers(0, W, nq), rng.integers(0, H, nq)], 1).astype(np.int32)
dxy = torch.from_numpy(xy).cuda()
dids = torch.zeros(nq * 16, dtype=torch.int32, device="cuda")
dw = torch.zeros(nq * 16, dtype=torch.float64, device="cuda")
dn = torch.zeros(nq, dtype=torch.int32, device="cuda")
args = (run, C.c_void_p(dxy.data_ptr()), C.c_size_t(nq), C.c_void_p(dids.data_ptr()), C.c_void_p(dw.data_ptr()),
        C.c_void_p(dn.data_ptr()))
G._call("fit_point_query", *args)
G._call("ctx_synchronize")
t0 = time.perf_counter()
for _ in range(5):
    G._call("fit_point_query", *args)
G._call("ctx_synchronize")
dt = (time.perf_counter() - t0) / 5
print(f"{nq} queries: {dt * 1e6:.1f} us per batch (wall, synchronized) -> {nq / dt / 1e9:.2f} G queries/s")
n = C.c_size_t()
nh = C.c_int()
sc = C.c_double()
G._call("fit_info", run, C.byref(n), C.byref(nh), C.byref(sc))
res = G._fit_collect(W, H, cfg, int(n.value), int(nh.value), float(sc.value),
                     lambda sv, fv, hist: G._call("fit_download", run, sv, fv, hist))
pick = rng.integers(0, nq, 1000)
ids, w, nn = G.pixel_weights_batch(res.sites, res.field, xy[pick])
gi = dids.cpu().numpy().reshape(nq, 16)[pick]
gw = dw.cpu().numpy().reshape(nq, 16)[pick]
gn = dn.cpu().numpy()[pick]
print("n match", np.array_equal(nn, gn), "ids match", np.array_equal(ids.view(np.int32), gi),
      "w max diff", float(np.abs(w - gw).max()), "mean n", float(gn.mean()))
