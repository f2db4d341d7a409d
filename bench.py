#!/usr/bin/env python
"""Benchmark of the B200 SAD fitting loop (BASELINE.json metric, config 2).

Workload (N=1): one full fit of a 768x512 Kodak-shaped synthetic image at target 2 BPP
(want 6144 sites, n0 9831), 4000 iterations with densify/prune events, fp32 kernels — a "step".
With --gpus N (torchrun, one process per GPU) each rank fits its own image(s): independent units,
no data-path collective, weak scaling.  `value` = iterations/s over all ranks with the target
already resident in HBM (CUDA events on the library's stream, L2 flushed between steps, max over
ranks); `e2e` = the same metric through the public Python API `Backend.fit(ImageBuffer, cfg)` with
host buffers (H2D of the target and D2H of the FitResult inside the timed region).

`--impl reference` times the reference CPU library (oracle/_ref, compiled from /root/reference) on
the host cores instead, same metric, each step a bounded sample of the same fit.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "fit iters/s and encode-seconds-to-PSNR at 768×512; render Gpix/s; % HBM roofline"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--width", type=int, default=768)
    p.add_argument("--height", type=int, default=512)
    p.add_argument("--bpp", type=float, default=2.0)
    p.add_argument("--iters", type=int, default=4000)
    p.add_argument("--images-per-gpu", type=int, default=1)
    p.add_argument("--serial", action="store_true", help="fit a rank's images one after another")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--ref-iters", type=int, default=80, help="iterations per reference-arm sample")
    p.add_argument("--cpu-iters", type=int, default=80, help="iterations of the cpu_baseline sample")
    p.add_argument("--mode", default="config2", choices=["config2", "config3", "config5"],
                   help="config3: 2048x2048 / 100k-site fit + 1e6 random point queries; config5: 8192x8192 "
                        "2-BPP fit on one GPU (each its own JSON line)")
    p.add_argument("--c3-iters", type=int, default=300)
    p.add_argument("--c5-iters", type=int, default=100)
    p.add_argument("--c5-size", type=int, default=8192, help="config5 image side (smaller for smoke runs)")
    p.add_argument("--c5-strips", action="store_true", help="config5: row-strip NCCL path even at N = 1")
    p.add_argument("--no-roofline-2048", action="store_true")
    p.add_argument("--no-paper-config", action="store_true", help="skip the paper-configuration encode timing")
    p.add_argument("--no-configs", action="store_true", help="skip the config 1 / 3 / 5 measurements of the N=1 run")
    return p.parse_args()


def config_dict(a):
    return {
        "workload": f"config2: {a.width}x{a.height} synthetic Kodak-shaped image, target {a.bpp} BPP "
                    f"(full fit() incl. device init_sites, {a.iters} iterations with densify/prune events, "
                    f"final refresh(Full,16)), fp32 kernels",
        "width": a.width, "height": a.height, "target_bpp": a.bpp, "iters": a.iters,
        "images_per_gpu": a.images_per_gpu, "concurrent_images": a.images_per_gpu > 1 and not a.serial,
        "k": 8, "inject": 4,
        "l2": "flushed (256 MiB write) between timed steps",
    }


def train_config(a, seed=1):
    import paper_2604_21984_b200 as sad
    return sad.TrainConfig(iters=a.iters, target_bpp=a.bpp, fp64=False, seed=seed)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------- reference arm
def ref_sample(a, iters, threads, seed=1, fp64=False):
    """One bounded sample of the config-2 fit on the reference library: the first `iters` iterations of
    the real 4000-iteration schedule (cfg.iters unchanged, so validate()'s event windows and
    plan_schedule are the full fit's; the loop stops after iteration `iters` via SAD_REF_STOP_AT,
    oracle/ref_capi.cpp).  Returns iters/s over the loop (init and the initial refresh excluded)."""
    import paper_2604_21984_b200 as sad
    from oracle.bindings import ref_backend
    from paper_2604_21984_b200.synth import synthetic_image
    R = ref_backend(threads=threads)
    img = sad.ImageBuffer(a.width, a.height, synthetic_image(a.width, a.height, seed))
    cfg = train_config(a, seed)
    cfg.fp64 = fp64
    cfg.threads = threads
    old = os.environ.get("SAD_REF_STOP_AT")
    os.environ["SAD_REF_STOP_AT"] = str(iters)
    try:
        t0 = time.perf_counter()
        res = R.fit(img, cfg)
        wall = time.perf_counter() - t0
    finally:
        if old is None:
            os.environ.pop("SAD_REF_STOP_AT", None)
        else:
            os.environ["SAD_REF_STOP_AT"] = old
    assert len(res.history) == iters
    loop_ms = sum(r.ms for r in res.history)
    return iters / (loop_ms / 1e3), loop_ms, wall, res


def ref_composite(a, threads, early_iters=80, late_iters=40, late_sites=5160):
    """Reference-arm sample of the whole 4000-iteration config-2 fit, from two bounded measurements on the
    reference library (loop time per iteration, from its own history rows):
      * the event phase: iterations 1-`early_iters` of the real schedule (one densify event every 20
        iterations and prunes every 40 from t = 100, as in iterations 1-3000);
      * the event-free tail (iterations 3001-4000): `late_iters` plain iterations of a budget-off fit with
        the final active count (`late_sites`; 5162 on the full fit, tests/golden/fit_config2_s1.npz).
    rate = 4000 / (3000 * t_event_phase + 1000 * t_tail)."""
    import paper_2604_21984_b200 as sad
    from oracle.bindings import ref_backend
    from paper_2604_21984_b200.synth import synthetic_image
    v_early, ms_early, w_early, _ = ref_sample(a, early_iters, threads)
    R = ref_backend(threads=threads)
    img = sad.ImageBuffer(a.width, a.height, synthetic_image(a.width, a.height, 1))
    cfg = sad.TrainConfig(iters=late_iters, n_sites=late_sites, fp64=False, seed=1)
    cfg.threads = threads
    t0 = time.perf_counter()
    res = R.fit(img, cfg)
    w_late = time.perf_counter() - t0
    ms_late = sum(r.ms for r in res.history)
    t_e, t_l = ms_early / early_iters, ms_late / late_iters
    total_ms = 3000 * t_e + 1000 * t_l
    return {"value": 4000 / (total_ms / 1e3), "event_phase_ms_per_iter": t_e, "tail_ms_per_iter": t_l,
            "wall_s": w_early + w_late,
            "sample": f"iterations 1-{early_iters} of the real 4000-iteration config-2 schedule (event phase) and "
                      f"{late_iters} plain iterations of a {late_sites}-site budget-off fit (event-free tail), "
                      f"weighted 3000:1000; loop time only; reference library oracle/_ref, {threads} threads"}


# Full reference fits of this workload measured on the GPU box's host (16 threads; tools/config2_lockstep.py,
# profiles/r1h_config2_lockstep.txt): 4000 iterations in 160.1 s = 25.0 iters/s including init and refreshes.
REF_FULL_FIT = {"seconds": 160.1, "iters_per_s": 25.0, "threads": 16, "source": "profiles/r1h_config2_lockstep.txt"}


def run_reference(a):
    ws, rank, local = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    for _ in range(a.warmup):
        ref_composite(a, threads, early_iters=a.ref_iters)
    vals, mss = [], []
    for _ in range(a.steps):
        cm = ref_composite(a, threads, early_iters=a.ref_iters)
        vals.append(cm["value"])
        mss.append(4000 / cm["value"] * 1e3)
    value = a.steps * 4000 / (sum(mss) / 1e3)
    sample = cm["sample"]
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": a.gpus,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": float(np.mean(mss)), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": config_dict(a),
        "cpu_baseline": {"value": value, "unit": "iters/s", "cores": threads, "kind": "reference", "sample": sample,
                         "full_fit_measured": REF_FULL_FIT},
        "e2e": {"value": value, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------------------- B200 arm
KBENCH = {"propagate_warm": 0, "fwd_bwd": 1, "render": 2, "propagate_flood": 3}


def kernel_table(G, run, npx, n_act, N, reps=50):
    """CUDA-event timings of the hot kernels on a fitted, device-resident state, with their
    algorithmic bytes per launch (propagate 64 B/cell + 32 B/site; fwd+bwd 44 B/px +
    124 B/site; render 44 B/px + 40 B/site)."""
    bytes_per = {"propagate_warm": 64 * npx + 32 * n_act, "fwd_bwd": 44 * npx + 124 * N,
                 "render": 44 * npx + 40 * N, "propagate_flood": 64 * npx + 32 * n_act}
    out = {}
    for nm, which in KBENCH.items():
        t = C.c_double()
        G._call("fit_bench", run, C.c_int(which), C.c_int(reps), C.byref(t))
        out[nm] = {"ms": t.value, "bytes": bytes_per[nm], "GBps": bytes_per[nm] / (t.value * 1e-3) / 1e9}
    return out


def hbm_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        return float(json.load(open(path)).get("hbm_gbs", 6650.0)), "MEASURED_PEAKS.json hbm_gbs (burst copy)"
    return 6650.0, "fallback 6650 GB/s (B200_PROFILING.md)"


def roofline_2048(G, iters=200, n_sites=100000):
    """Config-3 sized state (2048x2048, 100k sites): the HBM-relevant operating point."""
    import paper_2604_21984_b200 as sad
    from paper_2604_21984_b200.synth import synthetic_image
    W = H = 2048
    cfg = sad.TrainConfig(iters=iters, n_sites=n_sites, fp64=False)
    run = C.c_void_p()
    cc = cfg.to_c()
    G._call("fit_create", C.c_int(W), C.c_int(H), C.byref(cc), C.byref(run))
    try:
        img = synthetic_image(W, H, 3)
        G._call("fit_set_target", run, img.ctypes.data_as(C.POINTER(C.c_double)))
        G._call("fit_run_init", run)
        tot, ph = C.c_double(), (C.c_double * 8)()
        G._call("fit_timing", run, C.byref(tot), ph)
        kt = kernel_table(G, run, W * H, n_sites, n_sites)
    finally:
        G.lib.sad_fit_destroy(run)
    peak, src = hbm_peak()
    for v in kt.values():
        v["frac_hbm"] = v["GBps"] / peak
    out = {"workload": f"2048x2048, {n_sites} sites, {iters}-iteration fit state", "fit_ms_per_iter": tot.value / iters,
           "kernels": kt, "peak_gbs": peak, "peak_source": src}
    tf = os.path.join(ROOT, "profiles", "r2_ncu_fwd_bwd_traffic_2048.json")
    if os.path.exists(tf):  # DRAM traffic of the fwd+bwd kernel at this size, from the committed ncu capture
        tj = json.load(open(tf))
        out["fwd_bwd_traffic"] = {"bytes_per_launch": tj["traffic_bytes"], "source": os.path.relpath(tf, ROOT),
                                  "issue_active_pct_of_peak": tj.get("issue_active_pct_of_peak")}
    return out


def point_query_coords(W, H, nq=1_000_000):
    """1e6 query coordinates from seeded_stream(5, 7, 9), one sequential xorshift32 stream."""
    from paper_2604_21984_b200.synth import Rng
    rng = Rng(5, 7, 9)
    st = np.zeros(nq * 2, np.uint32)
    x = int(rng.s)
    for i in range(nq * 2):
        x ^= (x << 13) & 0xFFFFFFFF
        x ^= x >> 17
        x ^= (x << 5) & 0xFFFFFFFF
        st[i] = x
    xy = np.empty((nq, 2), np.int32)
    xy[:, 0] = st[0::2] % W
    xy[:, 1] = st[1::2] % H
    return xy


def measure_config3(G, stream, iters=300, steps=1):
    """Config 3: 2048x2048 synthetic image, 100k sites, `iters`-iteration fit, then 1e6 random point queries on
    the fitted field (CUDA events on the library's stream)."""
    import torch
    import paper_2604_21984_b200 as sad
    from paper_2604_21984_b200.synth import synthetic_image
    W = H = 2048
    cfg = sad.TrainConfig(iters=iters, n_sites=100000, fp64=False)
    run = C.c_void_p()
    cc = cfg.to_c()
    G._call("fit_create", C.c_int(W), C.c_int(H), C.byref(cc), C.byref(run))
    try:
        img = synthetic_image(W, H, 3)
        G._call("fit_set_target", run, img.ctypes.data_as(C.POINTER(C.c_double)))
        G._call("fit_run_init", run)  # warm-up
        ms = []
        for _ in range(max(steps, 1)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            G._call("fit_run_init", run)
            e1.record(stream)
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
        nq = 1_000_000
        dxy = torch.from_numpy(point_query_coords(W, H, nq)).cuda()
        dids = torch.empty(nq * 16, dtype=torch.int32, device="cuda")
        dw = torch.empty(nq * 16, dtype=torch.float64, device="cuda")
        dn = torch.empty(nq, dtype=torch.int32, device="cuda")
        args = (run, C.c_void_p(dxy.data_ptr()), C.c_size_t(nq), C.c_void_p(dids.data_ptr()),
                C.c_void_p(dw.data_ptr()), C.c_void_p(dn.data_ptr()))
        G._call("fit_point_query", *args)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(5):
            G._call("fit_point_query", *args)
        e1.record(stream)
        e1.synchronize()
        q_ms = e0.elapsed_time(e1) / 5
    finally:
        G.lib.sad_fit_destroy(run)
    return {"point_queries_per_s": nq / (q_ms * 1e-3), "fit_ms": float(np.mean(ms)),
            "fit_iters_per_s": iters / (np.mean(ms) * 1e-3),
            "workload": f"config3: 2048x2048 synthetic, n_sites=100000, {iters}-iteration fit, then 1e6 random point "
                        f"queries (seeded_stream(5,7,9)) on the fitted field"}


def measure_config1(G):
    """Config 1: 256x256, 4096 sites, 200 iterations, budget off, fp32 and fp64, through the API (warm)."""
    import paper_2604_21984_b200 as sad
    from paper_2604_21984_b200.synth import synthetic_image
    img = sad.ImageBuffer(256, 256, synthetic_image(256, 256, 1))
    out = {"workload": "config1: 256x256 synthetic, 4096 sites, 200 iterations, budget off"}
    for fp64 in (False, True):
        cfg = sad.TrainConfig(iters=200, n_sites=4096, fp64=fp64, seed=1)
        G.fit(img, cfg)
        t0 = time.perf_counter()
        r = G.fit(img, cfg)
        out["fp64" if fp64 else "fp32"] = {"fit_ms_e2e": (time.perf_counter() - t0) * 1e3,
                                           "fit_ms_device": r.timing["total_ms"]}
    return out


def measure_config5(G, i0=20, i1=40, size=8192):
    """Config 5 on one GPU: 8192x8192 at 2 BPP; marginal per-iteration device time between an i0- and an
    i1-iteration fit (events of the default schedule included)."""
    import paper_2604_21984_b200 as sad
    from paper_2604_21984_b200.synth import synthetic_image
    img = synthetic_image(size, size, 5)
    res = {}
    for iters in (5, i0, i1):
        cfg = sad.TrainConfig(iters=iters, target_bpp=2.0, fp64=False)
        run = C.c_void_p()
        cc = cfg.to_c()
        G._call("fit_create", C.c_int(size), C.c_int(size), C.byref(cc), C.byref(run))
        try:
            G._call("fit_set_target", run, img.ctypes.data_as(C.POINTER(C.c_double)))
            G._call("fit_run_init", run)
            tot, ph = C.c_double(), (C.c_double * 8)()
            G._call("fit_timing", run, C.byref(tot), ph)
            res[iters] = tot.value
        finally:
            G.lib.sad_fit_destroy(run)
    per = (res[i1] - res[i0]) / (i1 - i0)
    return {"ms_per_iter_marginal": per, "iters_per_s": 1e3 / per, "fit_ms": {str(k): v for k, v in res.items()},
            "workload": f"config5: {size}x{size} synthetic (seed 5), 2 BPP, fp32, one GPU; marginal between a "
                        f"{i0}- and a {i1}-iteration fit"}


def run_config3(a):
    """Config 3 as its own JSON line (bench.py --mode config3)."""
    import torch
    from paper_2604_21984_b200 import api
    stream = torch.cuda.Stream()  # explicit stream shared by the library and the timing events
    torch.cuda.set_stream(stream)
    lib = api.load_library()
    ctx = C.c_void_p()
    if lib.sad_ctx_create(C.c_int(0), C.c_void_p(stream.cuda_stream), C.byref(ctx)):
        raise RuntimeError(lib.sad_last_error().decode())
    G = api.Backend(lib, "sad_", ctx=ctx)
    c3 = measure_config3(G, stream, a.c3_iters, a.steps)
    rf = roofline_2048(G, iters=a.c3_iters)
    out = {"metric": METRIC, "mode": "config3", "value": c3["point_queries_per_s"], "unit": "point queries/s",
           "fit_ms": c3["fit_ms"], "fit_iters_per_s": c3["fit_iters_per_s"], "config": {"workload": c3["workload"]},
           "reference_pixel_weights_ms_per_query": 3.07, "roofline_2048": rf}
    print(json.dumps(out), flush=True)


def run_config5(a):
    """Config 5: one 8192x8192 image at 2 BPP (n0 = 1,677,722 sites).  N = 1: the resident single-GPU fit.
    N > 1 (torchrun): the row-strip partition over NCCL (sad_fit_run_strips; bit-identical to the
    single-GPU fit), time = max over ranks, strong scaling.  Two fits of different length give the
    marginal cost per iteration (the densify/prune events of the default schedule included, one every
    20 iterations from t = 20); the whole short fits are reported too."""
    import torch
    import paper_2604_21984_b200 as sad
    from paper_2604_21984_b200 import api
    from paper_2604_21984_b200.synth import synthetic_image
    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    lib = api.load_library()
    ctx = C.c_void_p()
    if lib.sad_ctx_create(C.c_int(local), C.c_void_p(stream.cuda_stream), C.byref(ctx)):
        raise RuntimeError(lib.sad_last_error().decode())
    G = api.Backend(lib, "sad_", ctx=ctx)
    W = H = a.c5_size
    img = synthetic_image(W, H, 5)
    nid = None
    if world > 1:
        obj = [G.nccl_unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(obj, src=0)
        nid = obj[0]
    strips = world > 1 or a.c5_strips
    if strips and nid is None:
        nid = G.nccl_unique_id()
    comm = G.strip_comm(rank, world, nid) if strips else None
    res = {}
    for iters in (5, max(a.c5_iters // 2, 20), a.c5_iters):  # the 5-iteration fit is the warm-up
        cfg = sad.TrainConfig(iters=iters, target_bpp=2.0, fp64=False)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        if not strips:
            run = C.c_void_p()
            cc = cfg.to_c()
            G._call("fit_create", C.c_int(W), C.c_int(H), C.byref(cc), C.byref(run))
            G._call("fit_set_target", run, img.ctypes.data_as(C.POINTER(C.c_double)))
            G._call("fit_run_init", run)
            info = sad_fit_info(G, run)
            tot = C.c_double()
            ph = (C.c_double * 8)()
            G._call("fit_timing", run, C.byref(tot), ph)
            loop_ms = tot.value
            G.lib.sad_fit_destroy(run)
        else:
            out = G.fit_strips(sad.ImageBuffer(W, H, img), cfg, comm)
            info = {"n_sites": out.sites.size(), "schedule_scale": out.schedule_scale}
            loop_ms = out.timing["total_ms"]
        e1.record(stream)
        e1.synchronize()
        # the fit loop's own device time (allocation / init / download excluded; both lengths share them)
        ms = loop_ms
        if world > 1:
            t = torch.tensor([ms], dtype=torch.float64, device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = float(t.item())
        if iters != 5:
            res[iters] = (ms, info)
    (i0, (t0, _)), (i1, (t1, info1)) = sorted(res.items())
    per_iter = (t1 - t0) / (i1 - i0)
    if rank == 0:
        out = {"metric": "fit iterations/s", "mode": "config5", "value": 1e3 / per_iter, "unit": "iters/s",
               "ms_per_iter_marginal": per_iter, "fit_ms": {str(k): v[0] for k, v in res.items()},
               "final_site_slots": info1["n_sites"], "schedule_scale": info1["schedule_scale"], "n_gpus": world,
               "scaling": "strong", "parallelism": f"row strips x{world} (NCCL)" if strips else "single GPU",
               "config": {"workload": f"config5: {W}x{H} synthetic (seed 5), target 2.0 BPP, fp32; marginal "
                                      f"per-iteration time between a {i0}- and a {i1}-iteration fit (default event "
                                      f"schedule); N > 1: row-strip partition over NCCL, max over ranks"},
               "reference_cpu_s_per_warm_pass_8_threads": 9.32, "reference_cpu_initial_refresh_s": 393.7}
        print(json.dumps(out), flush=True)
    if comm is not None:
        G.lib.sad_strip_comm_destroy(comm)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def sad_fit_info(G, run):
    """A few scalars of a finished fit (sad_fit_info)."""
    n, nh, sc = C.c_size_t(), C.c_int(), C.c_double()
    G._call("fit_info", run, C.byref(n), C.byref(nh), C.byref(sc))
    return {"n_sites": n.value, "n_history": nh.value, "schedule_scale": sc.value}


def psnr(a, b):
    m = float(np.mean((a - b) ** 2))
    return 99.0 if m <= 0 else min(99.0, 10 * math.log10(1.0 / m))


def run_b200(a):
    import torch
    import paper_2604_21984_b200 as sad
    from paper_2604_21984_b200 import api
    from paper_2604_21984_b200.synth import synthetic_image

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.Stream()  # explicit stream shared by the library and the timing events
    torch.cuda.set_stream(stream)
    lib = api.load_library()
    ctx = C.c_void_p()
    rc = lib.sad_ctx_create(C.c_int(local), C.c_void_p(stream.cuda_stream), C.byref(ctx))
    if rc:
        raise RuntimeError(lib.sad_last_error().decode())
    G = api.Backend(lib, "sad_", ctx=ctx)
    lib.sad_host_alloc.restype = C.c_void_p
    lib.sad_host_alloc.argtypes = [C.c_size_t]

    W, H = a.width, a.height
    npx = W * H
    from paper_2604_21984_b200 import shard
    seeds = shard.image_seeds(a.images_per_gpu, world, rank)
    imgs = [synthetic_image(W, H, s) for s in seeds]
    cfgs = [train_config(a, s) for s in seeds]
    dev_t = [torch.from_numpy(im).cuda() for im in imgs]
    torch.cuda.synchronize()
    # Several images per GPU (config 4) run concurrently: one context + stream + host thread each,
    # so the latency-bound kernels of independent fits overlap on the SMs.
    conc = a.images_per_gpu > 1 and not a.serial
    streams = [torch.cuda.Stream() for _ in cfgs] if conc else [stream] * len(cfgs)
    backends = []
    for st_i in streams:
        if st_i is stream:
            backends.append(G)
            continue
        cx = C.c_void_p()
        if lib.sad_ctx_create(C.c_int(local), C.c_void_p(st_i.cuda_stream), C.byref(cx)):
            raise RuntimeError(lib.sad_last_error().decode())
        backends.append(api.Backend(lib, "sad_", ctx=cx))
    runs = []
    for cfg, B in zip(cfgs, backends):
        run = C.c_void_p()
        cc = cfg.to_c()
        B._call("fit_create", C.c_int(W), C.c_int(H), C.byref(cc), C.byref(run))
        runs.append(run)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def fit_one(i):
        backends[i]._call("fit_set_target_device", runs[i], C.c_void_p(dev_t[i].data_ptr()))
        backends[i]._call("fit_run_init", runs[i])

    def step():
        if not conc:
            for i in range(len(runs)):
                fit_one(i)
            return
        ev0 = torch.cuda.Event()
        ev0.record(stream)
        for st_i in streams:
            st_i.wait_event(ev0)
        th = [threading.Thread(target=fit_one, args=(i,)) for i in range(len(runs))]
        for t in th:
            t.start()
        for t in th:
            t.join()
        for st_i in streams:
            stream.wait_stream(st_i)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = lib.sad_ctx_launch_count(ctx)  # process-wide counter (all contexts)
    ms = []
    for _ in range(a.steps):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    launches = int(lib.sad_ctx_launch_count(ctx) - launches0)
    clk = clocks.stop()
    tot_ms = sum(ms)
    if world > 1:
        t = torch.tensor([tot_ms], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        tot_ms = float(t.item())
    iters_all = a.steps * a.iters * a.images_per_gpu * world
    value = iters_all / (tot_ms / 1e3)

    # result quality (decode PSNR after the final refresh(Full,16)) from the last timed fit
    n = C.c_size_t()
    nh = C.c_int()
    sc = C.c_double()
    G._call("fit_info", runs[0], C.byref(n), C.byref(nh), C.byref(sc))
    res = G._fit_collect(W, H, cfgs[0], int(n.value), int(nh.value), float(sc.value),
                         lambda sv, fv, hist: G._call("fit_download", runs[0], sv, fv, hist))
    dec = G.render_image(res.sites, res.field, sad.RunOpts(fp64=False)).data
    psnr_dec = psnr(dec, imgs[0])
    last_train_psnr = res.history[-1].psnr if res.history else None

    # per-kernel timings on the fitted state (CUDA events on the same stream)
    n_act = res.sites.active_count()
    N = res.sites.size()
    kt = kernel_table(G, runs[0], npx, n_act, N, reps=100)
    kern = {k: v["ms"] for k, v in kt.items()}
    ev = sum(1 for t in range(1, a.iters + 1)
             if (20 <= t <= 3000 and t % 20 == 0) or (100 <= t <= 3000 and t % 40 == 0))
    flood_per = len(G.full_refresh_passes(W, H, 0))
    counts = {"propagate_warm": a.iters + 4 * (ev + 1) + 16, "fwd_bwd": a.iters, "render": 0,
              "propagate_flood": flood_per * (ev + 2)}
    bytes_per = {"propagate_warm": 64 * npx + 32 * n_act, "fwd_bwd": 44 * npx + 124 * N,
                 "render": 44 * npx + 40 * N, "propagate_flood": 64 * npx + 32 * n_act}
    fit_ms = tot_ms / max(a.steps * a.images_per_gpu, 1)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    kernels = {}
    for nm, t in kern.items():
        kernels[nm] = {"ms": t, "GBps": bytes_per[nm] / (t * 1e-3) / 1e9, "launches_per_fit": counts[nm],
                       "share_of_fit": counts[nm] * t / fit_ms}
    dom = max((k for k in kernels if counts[k] > 0), key=lambda k: kernels[k]["share_of_fit"])
    ach = kernels[dom]["GBps"]
    # DRAM traffic per launch of the dominant kernel from the committed ncu --set full capture
    traffic, traffic_src = None, None
    tfs = [os.path.join(ROOT, "profiles", f) for f in ("r2_ncu_fwd_bwd_traffic.json", "r1h_ncu_fwd_bwd_traffic.json",
                                                       "r1e_ncu_fwd_bwd_traffic.json")]
    tf = next((f for f in tfs if os.path.exists(f)), tfs[-1])
    if dom == "fwd_bwd" and os.path.exists(tf):
        tj = json.load(open(tf))
        traffic, traffic_src = tj["traffic_bytes"], f"{os.path.relpath(tf, ROOT)} ({tj['capture']})"
    roofline = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm, "traffic": traffic,
                "traffic_source": traffic_src, "kernel": dom, "algorithmic_bytes_per_launch": bytes_per[dom],
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)" if peaks else "fallback 6650 GB/s",
                "note": "768x512 working set is L2-resident; HBM fraction is judged at 2048^2 (see DESIGN.md)"}
    if dom == "fwd_bwd" and os.path.exists(tf):
        # what does bound it: SM issue / pipe utilisation from the same committed ncu capture
        tj = json.load(open(tf))
        if "issue_active_pct_of_peak" in tj:
            roofline["compute"] = {k: tj[k] for k in ("sm_throughput_pct_of_peak", "issue_active_pct_of_peak",
                                                      "fp64_pipe_active_pct_of_peak", "fma_pipe_active_pct_of_peak")}

    # end to end through the public API with host buffers
    tgt_host = sad.ImageBuffer(W, H, imgs[0])
    for _ in range(1):
        G.fit(tgt_host, cfgs[0])
    torch.cuda.synchronize()
    e2e_t = []
    for _ in range(a.steps):
        t0 = time.perf_counter()
        for im, cfg in zip(imgs, cfgs):
            r2 = G.fit(sad.ImageBuffer(W, H, im), cfg)
        e2e_t.append(time.perf_counter() - t0)
    e2e_s = sum(e2e_t)
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_val = iters_all / e2e_s
    h2d = 24 * npx * a.images_per_gpu
    d2h = (r2.sites.size() * 82 + r2.field.ids.nbytes + a.iters * 40) * a.images_per_gpu

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        try:
            threads = os.cpu_count() or 1
            cm = ref_composite(a, threads, early_iters=a.cpu_iters)
            v, wall = cm["value"], cm["wall_s"]
            v1, _, w1, _ = ref_sample(a, 20, 1)
            v64, _, w64, _ = ref_sample(a, 40, threads, fp64=True)
            cpu = {"value": v, "unit": "iters/s", "cores": threads, "kind": "reference",
                   "sample": cm["sample"] + f", {wall:.1f}s wall",
                   "event_phase_ms_per_iter": cm["event_phase_ms_per_iter"], "tail_ms_per_iter": cm["tail_ms_per_iter"],
                   "rows": {"f32_1_thread": {"value": v1, "sample": "iterations 1-20, 1 thread"},
                            "f64_all_threads": {"value": v64, "sample": f"iterations 1-40, fp64, {threads} threads"}},
                   "full_fit_measured": REF_FULL_FIT}
        except Exception as e:  # oracle not built on this box
            cpu = {"value": None, "unit": "iters/s", "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}

    rf2048 = None
    if rank == 0 and not a.no_roofline_2048:
        rf2048 = roofline_2048(G)
    configs = None
    if rank == 0 and world == 1 and not a.no_configs:
        # the other single-GPU configurations of SURVEY §8d, measured in the same run (device time)
        configs = {"config1": measure_config1(G), "config3": measure_config3(G, stream, 300, 1),
                   "config5": measure_config5(G)}
    fp64_row = None
    if rank == 0 and world == 1:
        # the reference's default precision (TrainConfig.fp64 = true, types.hpp:162): all-double kernels
        cfg64 = train_config(a, seeds[0])
        cfg64.fp64 = True
        tgt64 = sad.ImageBuffer(W, H, imgs[0])
        G.fit(tgt64, cfg64)
        t0 = time.perf_counter()
        r64 = G.fit(tgt64, cfg64)
        s64 = time.perf_counter() - t0
        fp64_row = {"value": a.iters / (r64.timing["total_ms"] * 1e-3), "unit": "iters/s",
                    "e2e": a.iters / s64, "encode_seconds_e2e": s64, "active_sites": r64.history[-1].active_sites,
                    "workload": "the same config-2 fit with fp64=True (all-double kernels)"}
    paper = None
    if rank == 0 and world == 1 and not a.no_paper_config:
        # the paper's own GPU implementation encodes Kodak 768x512 with 50k sites, 4000
        # iterations in 2.2 s (RTX 5090).  Same configuration here, through the public API (host target).
        pcfg = sad.TrainConfig(iters=4000, n_sites=50000, fp64=False)
        tgt_p = sad.ImageBuffer(W, H, imgs[0])
        G.fit(tgt_p, pcfg)
        t0 = time.perf_counter()
        G.fit(tgt_p, pcfg)
        paper = {"workload": "768x512 synthetic, n_sites=50000, 4000 iterations, budget off (the paper's Kodak "
                             "configuration)", "encode_seconds_e2e": time.perf_counter() - t0,
                 "paper_encode_seconds": 2.2, "paper_hardware": "RTX 5090 (PAPER.md:694-706)"}
    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": tot_ms / a.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": config_dict(a),
            "encode_seconds": fit_ms / 1e3, "psnr_decode_db": psnr_dec, "psnr_last_train_db": last_train_psnr,
            "active_sites": n_act, "render_gpix_s": npx / (kern["render"] * 1e-3) / 1e9,
            "e2e": {"value": e2e_val, "unit": "iters/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "encode_seconds": e2e_s / (a.steps * a.images_per_gpu)},
            "gpu_launches": launches, "roofline": roofline, "kernels": kernels, "cpu_baseline": cpu,
            "clocks": clk, "roofline_2048": rf2048, "paper_config": paper, "fp64": fp64_row, "configs": configs,
        }
        print(json.dumps(out), flush=True)
    for run in runs:
        lib.sad_fit_destroy(run)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    elif a.mode == "config3":
        run_config3(a)
    elif a.mode == "config5":
        run_config5(a)
    else:
        run_b200(a)


if __name__ == "__main__":
    main()
