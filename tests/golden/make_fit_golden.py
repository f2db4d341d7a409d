"""Generates the full-configuration fit goldens tests/golden/fit_*.npz from the compiled reference
(oracle/_ref/libsadref.so, the unmodified reference sources built by oracle/Makefile).  Run here, where
/root/reference exists; the GPU box only reads the committed files:

    python tests/golden/make_fit_golden.py [case ...]      (default: every case below)

Each case is one complete reference `fit` (the pre-warmed fit_impl replica, train.cpp:221-311, on all
host threads; results are thread-count invariant, test_train.cpp) of a synthetic image from
paper_2604_21984_b200.synth (the generator of SURVEY §8d).  Stored per case: the config, every history
row (loss, PSNR, active count), the schedule scale, SHA-256 digests of the final site arrays and of the
final candidate map, and the decode PSNR (fp32 render of the final field against the target).
tests/test_fit_configs.py runs the same fits on the GPU and requires all of it to be identical.
"""
import hashlib
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import numpy as np  # noqa: E402

import paper_2604_21984_b200 as sad  # noqa: E402
from oracle.bindings import ref_backend  # noqa: E402
from paper_2604_21984_b200.synth import synthetic_image  # noqa: E402

SITE_ARRAYS = ("x", "y", "log_tau", "radius", "col_r", "col_g", "col_b", "dir_x", "dir_y", "aniso", "active",
               "frozen")


def cases():
    """name -> (width, height, image seed, TrainConfig kwargs)."""
    out = {}
    for seed in range(1, 9):  # config 2: 768x512 Kodak-shaped, 2 BPP, 4000 iterations, events
        out[f"config2_s{seed}"] = (768, 512, seed, dict(iters=4000, target_bpp=2.0, fp64=False, seed=1))
    out["config2_fp64_s1"] = (768, 512, 1, dict(iters=4000, target_bpp=2.0, fp64=True, seed=1))
    # fp64 with the reference's default RunOpts::threads = 1 (types.hpp:163): the summation order the GPU's
    # fp64 path replays, on a second image
    out["config2_fp64_t1_s2"] = (768, 512, 2, dict(iters=4000, target_bpp=2.0, fp64=True, seed=1, threads=1))
    out["config2_fp64_s3"] = (768, 512, 3, dict(iters=4000, target_bpp=2.0, fp64=True, seed=1))
    out["config3_s1"] = (2048, 2048, 1, dict(iters=300, n_sites=100000, fp64=False, seed=1))
    out["config3_fp64_s1"] = (2048, 2048, 1, dict(iters=300, n_sites=100000, fp64=True, seed=1))
    # config 5 shape (8192^2, 2 BPP): 25 iterations, i.e. the initial refresh, one densify event (t = 20) with
    # its full re-seeded refresh, and the final refresh(Full, 16) (about 25 minutes on 8 host cores)
    out["config5_short_s5"] = (8192, 8192, 5, dict(iters=25, target_bpp=2.0, fp64=False, seed=1))
    return out


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def fit_record(res, target: sad.ImageBuffer, render) -> dict:
    rec = {
        "loss": np.array([r.loss for r in res.history], np.float64),
        "psnr": np.array([r.psnr for r in res.history], np.float64),
        "active": np.array([r.active_sites for r in res.history], np.int64),
        "schedule_scale": np.float64(res.schedule_scale),
        "n_sites": np.int64(res.sites.size()),
        "field_sha": digest(res.field.ids),
        "pass_index": np.int64(res.field.pass_index),
    }
    for p in SITE_ARRAYS:
        rec["sha_" + p] = digest(getattr(res.sites, p))
    img = render(res.sites, res.field)
    mse = float(np.mean((img - target.data) ** 2))
    rec["decode_psnr"] = np.float64(99.0 if mse <= 0 else 10.0 * np.log10(1.0 / mse))
    return rec


def main(names):
    threads = os.cpu_count() or 1
    R = ref_backend(threads=threads)
    todo = cases()
    for name in names or list(todo):
        w, h, seed, kw = todo[name]
        path = os.path.join(HERE, f"fit_{name}.npz")
        if os.path.exists(path):
            print(f"{name}: exists, skipped", flush=True)
            continue
        img = sad.ImageBuffer(w, h, synthetic_image(w, h, seed))
        cfg = sad.TrainConfig(**kw)
        nt = kw.get("threads", threads)
        cfg.threads = nt
        Rk = R if nt == threads else ref_backend(threads=nt)
        t0 = time.perf_counter()
        res = Rk.fit(img, cfg)
        sec = time.perf_counter() - t0
        rec = fit_record(res, img, lambda st, f: R.render_image(st, f, sad.RunOpts(fp64=False)).data)
        rec.update(width=np.int64(w), height=np.int64(h), image_seed=np.int64(seed), ref_seconds=np.float64(sec),
                   ref_threads=np.int64(nt), config=repr({k: v for k, v in kw.items() if k != "threads"}))
        np.savez_compressed(path, **rec)
        print(f"{name}: {len(res.history)} rows, active {res.history[-1].active_sites}, decode PSNR "
              f"{float(rec['decode_psnr']):.6f} dB, reference {sec:.1f} s on {nt} threads", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
