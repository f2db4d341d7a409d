"""Per-iteration exchange volume of the owner-merged row-strip fit (config 5 form) with R
virtual ranks on one device (loopback transport: same plans, same records as NCCL would move).
    python tools/strip_exchange.py [--size 8192] [--iters 40] [--world 8]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_21984_b200 as sad  # noqa: E402
from paper_2604_21984_b200.synth import synthetic_image  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=8192)
ap.add_argument("--iters", type=int, default=40)
ap.add_argument("--world", type=int, default=8)
ap.add_argument("--fp64", action="store_true", help="fp64: tagged tile records travel (reference-order strips)")
a = ap.parse_args()
G = sad.gpu_backend(0)
W = H = a.size
img = sad.ImageBuffer(W, H, synthetic_image(W, H, 5))
cfg = sad.TrainConfig(iters=a.iters, target_bpp=2.0, fp64=a.fp64)
t0 = time.perf_counter()
outs = G.fit_strips_loopback(img, cfg, a.world)
wall = time.perf_counter() - t0
ref = G.fit(img, cfg)
same = all([sad.history_line(r) for r in o.history] == [sad.history_line(r) for r in ref.history] for o in outs)
n = ref.sites.size()
R = a.world
rec = 192  # bytes per owner record (id + 11 double-doubles)
sent = [o.timing["records_sent"] for o in outs]
per_iter_records = [s / a.iters for s in sent]
param_bytes = 80 * n * (R - 1) / R  # received per rank per iteration (parameter all-gather)
halo_bytes = 2 * W * 32 * 2  # one warm pass: one row above and below, sent and received
out = {"image": f"{W}x{H}", "fp64": a.fp64, "world": R, "iters": a.iters, "sites": n, "identical_to_single_gpu": same,
       "records_sent_per_rank_per_iter": per_iter_records,
       "owner_record_bytes_per_rank_per_iter_max": max(per_iter_records) * rec,
       "param_allgather_bytes_per_rank_per_iter": param_bytes,
       "halo_bytes_per_rank_per_warm_pass": halo_bytes,
       "old_dense_allgather_bytes_per_rank_per_iter": 160 * n * R,
       "loopback_wall_s": wall}
print(json.dumps(out))
