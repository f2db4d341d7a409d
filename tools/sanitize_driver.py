"""Every kernel of the library once or twice at small sizes, each result checked against the CPU oracle.
Run it under compute-sanitizer where that is available, and with the bound-checked build
(SAD_LIB=paper_2604_21984_b200/libsad_b200_checked.so) everywhere: it then also reports the kernels'
bound-check failures (tests/test_checked_build.py).

    SAD_LIB=paper_2604_21984_b200/libsad_b200_checked.so python tools/sanitize_driver.py
    compute-sanitizer --tool racecheck python tools/sanitize_driver.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2604_21984_b200 as sad  # noqa: E402
from oracle.bindings import c_backend, have_ref, ref_backend  # noqa: E402
from tests.fixtures import random_model, random_sites, random_target, synth_target  # noqa: E402

G = sad.gpu_backend(0)
R = ref_backend() if have_ref() else c_backend()
F32, F64 = sad.RunOpts(fp64=False), sad.RunOpts(fp64=True)
checks = []


def check(name, ok):
    checks.append((name, bool(ok)))
    print(f"{name}: {'ok' if ok else 'MISMATCH'}", flush=True)


w, h = 48, 40
st = random_model(w, h, 70, 3)
st.deactivate(5)
tgt = random_target(w, h, 4)
for opts in (F32, F64):
    fg, fr = sad.CandidateField(), sad.CandidateField()
    fg.resize(w, h, 8)
    fr.resize(w, h, 8)
    G.refresh(st, fg, sad.RefreshMode.Full, 4, 4, 7, opts)
    R.refresh(st, fr, sad.RefreshMode.Full, 4, 4, 7, opts)
    G.refresh(st, fg, sad.RefreshMode.WarmStart, 2, 4, 8, opts)
    R.refresh(st, fr, sad.RefreshMode.WarmStart, 2, 4, 8, opts)
    check(f"refresh fp64={opts.fp64}", np.array_equal(fg.ids, fr.ids))
    check(f"render fp64={opts.fp64}", np.array_equal(G.render_image(st, fg, opts).data, R.render_image(st, fr, opts).data))
    for rem in (False, True):
        gg, gr = sad.GradBuffer(), sad.GradBuffer()
        lg = G.backward_image(st, fg, tgt, gg, opts, rem)
        lr = R.backward_image(st, fr, tgt, gr, opts, rem)
        check(f"backward fp64={opts.fp64} removal={rem}", lg == lr and np.array_equal(gg.data, gr.data))
    dl = random_target(w, h, 5)
    gg, gr = sad.GradBuffer(), sad.GradBuffer()
    G.backward_pixel_grad(st, fg, dl, gg, opts)
    R.backward_pixel_grad(st, fr, dl, gr, opts)
    check(f"pixel_grad fp64={opts.fp64}", np.array_equal(gg.data[:, :10], gr.data[:, :10]))
    check(f"image_loss fp64={opts.fp64}", G.image_loss(st, fg, tgt, opts) == R.image_loss(st, fr, tgt, opts))
# K = 16 and cell = 2 instantiations
for k, cell in ((16, 1), (5, 2)):
    fg, fr = sad.CandidateField(), sad.CandidateField()
    fg.resize(w, h, k, cell)
    fr.resize(w, h, k, cell)
    G.refresh(st, fg, sad.RefreshMode.Full, 3, 4, 9, F32)
    R.refresh(st, fr, sad.RefreshMode.Full, 3, 4, 9, F32)
    check(f"refresh k={k} cell={cell}", np.array_equal(fg.ids, fr.ids))
f = sad.CandidateField()
f.resize(w, h, 8)
R.refresh(st, f, sad.RefreshMode.Full, 4, 4, 7, F64)
sg, sr = G.accumulate_stats(st, f, tgt), R.accumulate_stats(st, f, tgt)
check("stats", np.array_equal(sg.data, sr.data))
pix = np.stack([np.arange(0, w, 3), np.arange(0, w, 3) % h], 1)
ig, wg, ng = G.pixel_weights_batch(st, f, pix)
ir, wr, nr = R.pixel_weights_batch(st, f, pix)
check("pixel_weights", np.array_equal(ig, ir) and np.array_equal(wg, wr))
check("render_id_map", np.array_equal(G.render_id_map(st, f), R.render_id_map(st, f)))
check("exact_topk", np.array_equal(G.exact_topk_batch(st, pix, 8, sad.normalization_scale(w, h), False),
                                   R.exact_topk_batch(st, pix, 8, sad.normalization_scale(w, h), False)))
a, b = st.copy(), st.copy()
ga = sad.GradBuffer(st.size())
ga.data[:] = np.random.default_rng(1).normal(size=ga.data.shape) * 1e-3
ma, mb = sad.AdamState(st.size()), sad.AdamState(st.size())
G.adam_step(a, ga, ma, w, h, sad.TrainConfig())
R.adam_step(b, ga, mb, w, h, sad.TrainConfig())
check("adam", np.array_equal(a.x, b.x) and np.array_equal(ma.v, mb.v))
G.clamp_project(a, w, h, sad.TrainConfig())
R.clamp_project(b, w, h, sad.TrainConfig())
check("clamp", np.array_equal(a.x, b.x))
a, b = st.copy(), st.copy()
check("prune", G.prune(a, sr, 0.2) == R.prune(b, sr, 0.2) and np.array_equal(a.active, b.active))
ma, mb = sad.AdamState(a.size()), sad.AdamState(b.size())
check("densify", G.densify(a, ma, sr, tgt, 0.5, sad.TrainConfig()) == R.densify(b, mb, sr, tgt, 0.5, sad.TrainConfig())
      and np.array_equal(a.x, b.x))
i1, i2 = sad.SiteStore(), sad.SiteStore()
img = synth_target(64, 48, 2)
G.init_sites(i1, img, 90, sad.TrainConfig())
R.init_sites(i2, img, 90, sad.TrainConfig())
check("init_sites", np.array_equal(i1.x, i2.x))
g = sad.GradBuffer(st.size())
g.data[:] = np.random.default_rng(2).normal(size=g.data.shape)
g2 = sad.GradBuffer(st.size())
g2.data[:] = g.data
G.tau_diffusion(st, f, 0.3, g)
R.tau_diffusion(st, f, 0.3, g2)
check("tau_diffusion", np.array_equal(g.data, g2.data))
# resident fits: plain iterations (graphs), events (stats, prune, densify, refresh), fp32 and fp64
for fp64 in (False, True):
    cfg = sad.TrainConfig(iters=45, target_bpp=3.0, fp64=fp64, seed=2, densify_start=10, densify_every=10,
                          prune_start=20, prune_every=20, tau_diffusion_lambda=0.2 if not fp64 else 0.0)
    fa, fb = G.fit(img, cfg), R.fit(img, cfg)
    check(f"fit fp64={fp64}", [sad.history_line(r) for r in fa.history] == [sad.history_line(r) for r in fb.history])
# codec decode render
data = G.encode_sites(fa.sites, 64, 48)
dimg, _ = G.decode_render(data)
rimg, _ = R.decode_render(data)
check("decode_render", np.array_equal(dimg.data, rimg.data))
# strips (loopback virtual ranks)
cfg = sad.TrainConfig(iters=25, target_bpp=3.0, fp64=False, seed=3, densify_start=10, densify_every=10)
single = G.fit(img, cfg)
parts = G.fit_strips_loopback(img, cfg, 2)
check("strips", all([sad.history_line(r) for r in p.history] == [sad.history_line(r) for r in single.history]
                    for p in parts))
cfg64 = sad.TrainConfig(iters=25, target_bpp=3.0, fp64=True, seed=3, densify_start=10, densify_every=10)
single64 = G.fit(img, cfg64)
parts64 = G.fit_strips_loopback(img, cfg64, 2)  # fp64: tagged records shipped to the owners (ordered strips)
check("strips fp64", all([sad.history_line(r) for r in p.history] == [sad.history_line(r) for r in single64.history]
                         for p in parts64))
bad = [n for n, ok in checks if not ok]
fails = int(G.lib.sad_debug_check_failures())  # -1: product build (no bound checks compiled in)
print(f"{len(checks)} checks, {len(bad)} mismatches {bad}; kernel bound-check failures: {fails}")
sys.exit(1 if bad or fails > 0 else 0)
