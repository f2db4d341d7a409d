"""Full config-2 lockstep: the GPU fit and the compiled reference's fit (all host threads) of the same
768x512 synthetic image at 2 BPP, 4000 iterations with events.  Prints whether every history line
(%.17g loss / PSNR, active count), the final sites and the final candidate map are identical, the decode
PSNR of both, and the full-fit wall times.   python tools/config2_lockstep.py [seed ...]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_21984_b200 as sad  # noqa: E402
from oracle.bindings import ref_backend  # noqa: E402
from paper_2604_21984_b200.synth import synthetic_image  # noqa: E402

threads = os.cpu_count() or 1
G = sad.gpu_backend(0)
R = ref_backend(threads=threads)
# config 3 instead: python tools/config2_lockstep.py --config3 [seed]  (2048^2, 100k sites, 300 iterations)
C3 = "--config3" in sys.argv
args = [a for a in sys.argv[1:] if not a.startswith("--")]
W, H = (2048, 2048) if C3 else (768, 512)
ITERS = 300 if C3 else 4000


def make_cfg():
    if C3:
        return sad.TrainConfig(iters=ITERS, n_sites=100000, fp64=False, seed=1)
    return sad.TrainConfig(iters=ITERS, target_bpp=2.0, fp64=False, seed=1)


for seed in [int(x) for x in args] or [1]:
    img = sad.ImageBuffer(W, H, synthetic_image(W, H, seed))
    cfg = make_cfg()
    G.fit(img, cfg)  # warm (graph capture, allocation)
    t0 = time.perf_counter()
    a = G.fit(img, cfg)
    tg = time.perf_counter() - t0
    cfg_r = make_cfg()
    cfg_r.threads = threads
    t0 = time.perf_counter()
    b = R.fit(img, cfg_r)
    tr = time.perf_counter() - t0
    la = [sad.history_line(r) for r in a.history]
    lb = [sad.history_line(r) for r in b.history]
    first = next((i for i, (x, y) in enumerate(zip(la, lb)) if x != y), None)
    same_sites = all(np.array_equal(getattr(a.sites, p), getattr(b.sites, p))
                     for p in ("x", "y", "log_tau", "radius", "col_r", "col_g", "col_b", "dir_x", "dir_y", "aniso",
                               "active"))
    pa = G.render_image(a.sites, a.field, sad.RunOpts(fp64=False)).data
    pb = R.render_image(b.sites, b.field, sad.RunOpts(fp64=False)).data

    def psnr(x):
        m = float(np.mean((x - img.data) ** 2))
        return 99.0 if m <= 0 else 10 * np.log10(1.0 / m)

    print(f"{W}x{H} seed {seed}: history {f'identical ({ITERS} lines)' if first is None else f'first difference at iter {first + 1}'}; "
          f"final sites identical {same_sites}; final map identical {np.array_equal(a.field.ids, b.field.ids)}; "
          f"decode PSNR gpu {psnr(pa):.6f} ref {psnr(pb):.6f}; active {a.history[-1].active_sites}; "
          f"fit wall gpu {tg:.3f} s (e2e), reference {tr:.1f} s on {threads} threads ({ITERS / tr:.2f} iters/s)",
          flush=True)
