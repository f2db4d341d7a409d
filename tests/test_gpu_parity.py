"""GPU parity tests: the CUDA path (libsad_b200.so through the C ABI) against the CPU oracle on the
same seeded inputs.  Oracle = the compiled reference library when present (oracle/_ref/libsadref.so,
prebuilt here and shipped with the repo), else the plain-C restatement pinned to it by
tests/test_oracle.py.

Tolerances (BASELINE.json north_star): top-K maps identical; rendered pixels and site gradients
within 1e-5 relative (per-slot L2 norm for gradients); loss within 1e-7 relative.
The float path is built to be bit-exact, so most tests also report / assert exact equality.
"""
import numpy as np
import pytest

import paper_2604_21984_b200 as sad
from oracle.bindings import c_backend, have_ref, ref_backend
from tests.fixtures import random_model, random_sites, random_target, ramp_image, synth_target

pytestmark = pytest.mark.gpu

F32 = sad.RunOpts(fp64=False)
F64 = sad.RunOpts(fp64=True)


@pytest.fixture(scope="module")
def G():
    return sad.gpu_backend(0)


@pytest.fixture(scope="module")
def R():
    return ref_backend() if have_ref() else c_backend()


def _field(w, h, k=8, cell=1):
    f = sad.CandidateField()
    f.resize(w, h, k, cell)
    return f


def _render_ok(a, b):
    return np.all(np.abs(a - b) <= 1e-5 * np.maximum(np.abs(b), 1e-3))


def _grad_ok(g, r, slots=11):
    for k in range(slots):
        d = np.linalg.norm(g[:, k] - r[:, k])
        n = np.linalg.norm(r[:, k])
        assert d <= 1e-5 * n or d == 0.0, f"slot {k}: rel {d / max(n, 1e-300)}"


# ---------------------------------------------------------------------------- candidates
@pytest.mark.parametrize("fp64", [False, True])
@pytest.mark.parametrize("case", [(24, 16, 40, 99), (64, 48, 120, 5), (96, 64, 200, 55), (37, 29, 60, 8)])
def test_refresh_maps_identical(G, R, fp64, case):
    w, h, n, seed = case
    opts = sad.RunOpts(fp64=fp64)
    st = random_sites(w, h, n, seed)
    st.deactivate(3)
    fg, fr = _field(w, h), _field(w, h)
    G.refresh(st, fg, sad.RefreshMode.Full, 4, 4, 1234, opts)
    R.refresh(st, fr, sad.RefreshMode.Full, 4, 4, 1234, opts)
    assert np.array_equal(fg.ids, fr.ids)
    assert fg.pass_index == fr.pass_index and fg.synced_generation == st.generation
    G.refresh(st, fg, sad.RefreshMode.WarmStart, 3, 4, 77, opts)
    R.refresh(st, fr, sad.RefreshMode.WarmStart, 3, 4, 77, opts)
    assert np.array_equal(fg.ids, fr.ids)


def test_propagate_pass_box_step(G, R):
    """test_candidates.cpp:122-168 setup: Box3 step-2 pass after two warm passes."""
    st = random_sites(24, 16, 40, 99)
    fg, fr = _field(24, 16), _field(24, 16)
    G.jfa_seed(st, fg)
    R.jfa_seed(st, fr)
    assert np.array_equal(fg.ids, fr.ids)
    for B in (G, R):
        f = fg if B is G else fr
        B.refresh(st, f, sad.RefreshMode.WarmStart, 2, 4, 1234, sad.RunOpts())
        B.propagate_pass(st, f, sad.PassSpec(2, sad.Stencil.Box3), 4, 777, sad.RunOpts())
    assert np.array_equal(fg.ids, fr.ids)


@pytest.mark.parametrize("stencil,step", [(sad.Stencil.Axial, 1), (sad.Stencil.Box3, 4), (sad.Stencil.Box3, 1)])
def test_propagate_fallback_cells(G, R, stencil, step):
    """Own lists holding a repeated id take the K=8 kernels' exact streaming fallback; the map must
    still equal the reference's first-appearance pool result (candidates.cpp:108-135)."""
    w, h = 40, 32
    st = random_sites(w, h, 80, 17)
    fg, fr = _field(w, h), _field(w, h)
    G.refresh(st, fg, sad.RefreshMode.Full, 2, 4, 5, F32)
    R.refresh(st, fr, sad.RefreshMode.Full, 2, 4, 5, F32)
    assert np.array_equal(fg.ids, fr.ids)
    ids = fg.ids.reshape(-1, 8).copy()
    rows = np.random.default_rng(3).choice(ids.shape[0], 300, replace=False)
    full = rows[ids[rows, 3] != sad.CandidateField.kEmpty]
    ids[full, 3] = ids[full, 0]
    ids[rows[:40], 1] = ids[rows[:40], 0]
    fg.ids = ids.reshape(-1).copy()
    fr.ids = ids.reshape(-1).copy()
    for B, f in ((G, fg), (R, fr)):
        B.propagate_pass(st, f, sad.PassSpec(step, stencil), 4, 31, F32)
    assert np.array_equal(fg.ids, fr.ids)


def test_propagate_nan_site(G, R):
    """A site with a NaN coordinate gives NaN logits (no order); cells that see it are recomputed
    in the reference's feed order, and the rest of the map is unaffected."""
    w, h = 40, 32
    st = random_sites(w, h, 80, 23)
    fg, fr = _field(w, h), _field(w, h)
    G.refresh(st, fg, sad.RefreshMode.Full, 2, 4, 5, F32)
    R.refresh(st, fr, sad.RefreshMode.Full, 2, 4, 5, F32)
    st.x[11] = np.nan
    st.bump()
    for B, f in ((G, fg), (R, fr)):
        B.propagate_pass(st, f, sad.PassSpec(1, sad.Stencil.Axial), 4, 31, F32)
        B.propagate_pass(st, f, sad.PassSpec(2, sad.Stencil.Box3), 4, 32, F32)
    assert np.array_equal(fg.ids, fr.ids)


@pytest.mark.parametrize("k,cell", [(1, 1), (3, 1), (12, 1), (16, 1), (8, 2), (5, 3)])
def test_refresh_other_k_and_cell(G, R, k, cell):
    st = random_model(40, 30, 70, 4)
    fg, fr = _field(40, 30, k, cell), _field(40, 30, k, cell)
    G.refresh(st, fg, sad.RefreshMode.Full, 3, 5, 9, F32)
    R.refresh(st, fr, sad.RefreshMode.Full, 3, 5, 9, F32)
    assert np.array_equal(fg.ids, fr.ids)


def test_jfa_seed_collisions(G, R):
    """test_candidates.cpp:97-120 plus many forced collisions (two sites per cell)."""
    st = sad.SiteStore()
    st.append(sad.Site(x=10.3, y=5.2, radius=1.0, log_tau=4.0))
    st.append(sad.Site(x=10.45, y=4.8, radius=6.0, log_tau=4.0))
    rng = np.random.default_rng(1)
    for i in range(400):
        cx, cy = rng.integers(0, 32, 2)
        for _ in range(2):
            st.append(sad.Site(x=cx + rng.uniform(-0.49, 0.49), y=cy + rng.uniform(-0.49, 0.49),
                               radius=rng.uniform(1, 6), log_tau=rng.uniform(3, 9)))
    fg, fr = _field(32, 32), _field(32, 32)
    G.jfa_seed(st, fg)
    R.jfa_seed(st, fr)
    assert np.array_equal(fg.ids, fr.ids)


def test_inject_only_empty_field(G, R):
    st = random_sites(40, 40, 80, 77)
    for seed in (1000, 1001):
        fg, fr = _field(40, 40), _field(40, 40)
        G.refresh(st, fg, sad.RefreshMode.WarmStart, 1, 4, seed, F32)
        R.refresh(st, fr, sad.RefreshMode.WarmStart, 1, 4, seed, F32)
        assert np.array_equal(fg.ids, fr.ids)


# ---------------------------------------------------------------------------- render / backward
@pytest.mark.parametrize("fp64", [False, True])
def test_render_matches(G, R, fp64):
    opts = sad.RunOpts(fp64=fp64)
    st = random_model(64, 48, 90, 7)
    f = _field(64, 48)
    R.refresh(st, f, sad.RefreshMode.Full, 4, 4, 7, opts)
    a = G.render_image(st, f, opts).data
    b = R.render_image(st, f, opts).data
    assert _render_ok(a, b)
    assert np.array_equal(a, b), f"render not bit-exact: {np.count_nonzero(a != b)} differ"


@pytest.mark.parametrize("fp64", [False, True])
@pytest.mark.parametrize("removal", [False, True])
def test_backward_matches(G, R, fp64, removal):
    opts = sad.RunOpts(fp64=fp64)
    st = random_model(64, 64, 50, 100)
    tgt = random_target(64, 64, 200)
    f = _field(64, 64)
    R.refresh(st, f, sad.RefreshMode.Full, 4, 4, 7, opts)
    gg, gr = sad.GradBuffer(), sad.GradBuffer()
    lg = G.backward_image(st, f, tgt, gg, opts, removal)
    lr = R.backward_image(st, f, tgt, gr, opts, removal)
    assert abs(lg - lr) <= 1e-7 * abs(lr)
    _grad_ok(gg.data, gr.data)
    assert gg.nonfinite == gr.nonfinite
    # both precisions are bit-identical (fp64 through the device glibc-exp port)
    assert lg == lr
    assert np.array_equal(gg.data, gr.data)


@pytest.mark.parametrize("w,h,k,cell", [(37, 29, 1, 1), (37, 29, 3, 1), (50, 34, 8, 1), (40, 30, 12, 1),
                                         (40, 30, 16, 2), (23, 17, 5, 3)])
def test_tiles_ragged_and_other_k(G, R, w, h, k, cell):
    """The fp32 two-lanes-per-pixel backward and stats kernels on image sizes that are not multiples of
    their 16x8 / 8x8 tiles, with lists shorter than 8 (lane 1 partly or wholly past the list end) and
    K = 16 (the 16-slot instantiations).  fp32 loss and gradients must be bit-identical."""
    st = random_model(w, h, 45, 17 + k)
    st.deactivate(2)
    tgt = random_target(w, h, 5 + k)
    f = _field(w, h, k, cell)
    R.refresh(st, f, sad.RefreshMode.Full, 3, 4, 11, F32)
    for removal in (False, True):
        gg, gr = sad.GradBuffer(), sad.GradBuffer()
        lg = G.backward_image(st, f, tgt, gg, F32, removal)
        lr = R.backward_image(st, f, tgt, gr, F32, removal)
        assert lg == lr
        assert np.array_equal(gg.data, gr.data)
        assert gg.nonfinite == gr.nonfinite
    dl = random_target(w, h, 3)
    dl.data -= 0.5
    gg, gr = sad.GradBuffer(), sad.GradBuffer()
    G.backward_pixel_grad(st, f, dl, gg, F32)
    R.backward_pixel_grad(st, f, dl, gr, F32)
    assert np.array_equal(gg.data[:, :10], gr.data[:, :10])
    assert G.image_loss(st, f, tgt, F32) == R.image_loss(st, f, tgt, F32)
    assert np.array_equal(G.render_image(st, f, F32).data, R.render_image(st, f, F32).data)
    assert np.array_equal(G.render_id_map(st, f), R.render_id_map(st, f))
    sg = G.accumulate_stats(st, f, tgt)
    sr = R.accumulate_stats(st, f, tgt)
    assert sg.valid_pixels == sr.valid_pixels
    assert np.array_equal(sg.data, sr.data)


@pytest.mark.parametrize("w,h,k,cell", [(37, 29, 1, 1), (50, 34, 8, 1), (40, 30, 16, 2), (23, 17, 5, 3)])
def test_fp64_ordered_ragged_and_other_k(G, R, w, h, k, cell):
    """The fp64 reference-order backward (16x16 reference tiles, TileReducer replay) on ragged image
    sizes, short lists, K = 16 and coarse cells: loss, every gradient channel (with and without the
    removal delta, and the adjoint entry point) and the non-finite count bit-identical."""
    st = random_model(w, h, 45, 31 + k)
    st.deactivate(3)
    tgt = random_target(w, h, 9 + k)
    f = _field(w, h, k, cell)
    R.refresh(st, f, sad.RefreshMode.Full, 3, 4, 11, F64)
    for removal in (False, True):
        gg, gr = sad.GradBuffer(), sad.GradBuffer()
        assert G.backward_image(st, f, tgt, gg, F64, removal) == R.backward_image(st, f, tgt, gr, F64, removal)
        assert np.array_equal(gg.data, gr.data)
        assert gg.nonfinite == gr.nonfinite
    dl = random_target(w, h, 4)
    dl.data -= 0.5
    gg, gr = sad.GradBuffer(), sad.GradBuffer()
    G.backward_pixel_grad(st, f, dl, gg, F64)
    R.backward_pixel_grad(st, f, dl, gr, F64)
    assert np.array_equal(gg.data[:, :10], gr.data[:, :10])


@pytest.mark.parametrize("k", [5, 8, 12])
def test_pixel_weights_batch(G, R, k):
    """pixel_weights (render.cpp:92-104) batched: per query the kept ids in list order and their double
    softmax weights, bit-identical (device port of glibc's exp)."""
    w, h = 45, 37
    st = random_model(w, h, 60, 29)
    st.deactivate(4)
    f = _field(w, h, k)
    R.refresh(st, f, sad.RefreshMode.Full, 3, 4, 13, F32)
    rng = np.random.default_rng(k)
    pix = np.stack([rng.integers(0, w, 300), rng.integers(0, h, 300)], 1)
    ig, wg, ng = G.pixel_weights_batch(st, f, pix)
    ir, wr, nr = R.pixel_weights_batch(st, f, pix)
    assert np.array_equal(ng, nr)
    assert np.array_equal(ig, ir)
    # all-double softmax through the device glibc-exp port: bit-identical
    assert np.array_equal(wg.view(np.uint64), wr.view(np.uint64))


def test_pixel_weights_short_lists(G, R):
    """Point queries on lists that end in sentinels (6 sites, K=8) and hold an inactive site: the
    eight-lanes-per-query kernel keeps the reference's break-at-sentinel / skip-inactive rules, every
    pixel of the image, bit-identical; out-of-range queries are refused as in the reference."""
    w, h = 33, 29
    st = random_model(w, h, 6, 41)
    st.deactivate(2)
    f = _field(w, h, 8)
    R.refresh(st, f, sad.RefreshMode.Full, 2, 4, 17, F32)
    assert (f.ids.reshape(-1, 8) == 0xFFFFFFFF).any()
    yy, xx = np.mgrid[0:h, 0:w]
    pix = np.stack([xx.ravel(), yy.ravel()], 1)
    ig, wg, ng = G.pixel_weights_batch(st, f, pix)
    ir, wr, nr = R.pixel_weights_batch(st, f, pix)
    assert np.array_equal(ng, nr) and np.array_equal(ig, ir)
    assert np.array_equal(wg.view(np.uint64), wr.view(np.uint64))
    # the branch-free render (masked slots add +0.0) on the same short lists
    assert np.array_equal(G.render_image(st, f, F32).data, R.render_image(st, f, F32).data)
    for q in ([w, 0], [-1, 3], [0, h]):  # the reference's std::invalid_argument (render.cpp:95-96)
        with pytest.raises(sad.api.InvalidArgument):
            G.pixel_weights_batch(st, f, np.array([q]))


def test_loss_identity_and_pixgrad(G, R):
    """test_grad.cpp:116-128: image_loss == backward loss; adjoint entry point parity."""
    st = random_model(64, 64, 60, 7)
    tgt = random_target(64, 64, 8)
    f = _field(64, 64)
    R.refresh(st, f, sad.RefreshMode.Full, 4, 4, 7, F32)
    l1 = G.image_loss(st, f, tgt, F32)
    l2 = G.backward_image(st, f, tgt, sad.GradBuffer(), F32)
    assert l1 == l2 == R.image_loss(st, f, tgt, F32)
    dl = random_target(64, 64, 9)
    dl.data -= 0.5
    gg, gr = sad.GradBuffer(), sad.GradBuffer()
    G.backward_pixel_grad(st, f, dl, gg, F32)
    R.backward_pixel_grad(st, f, dl, gr, F32)
    _grad_ok(gg.data, gr.data, 10)


def test_backward_synth_image_large(G, R):
    """A realistic field: fitted-size synthetic image, 2k sites, fp32 path."""
    w, h = 256, 192
    tgt = synth_target(w, h, 3)
    st = sad.SiteStore()
    R.init_sites(st, tgt, 2000, sad.TrainConfig())
    f = _field(w, h)
    R.refresh(st, f, sad.RefreshMode.Full, 4, 4, 1, F32)
    fg = _field(w, h)
    G.refresh(st, fg, sad.RefreshMode.Full, 4, 4, 1, F32)
    assert np.array_equal(f.ids, fg.ids)
    gg, gr = sad.GradBuffer(), sad.GradBuffer()
    assert G.backward_image(st, f, tgt, gg, F32, False) == R.backward_image(st, f, tgt, gr, F32, False)
    _grad_ok(gg.data, gr.data, 10)


def test_stale_and_empty_errors(G):
    st = random_model(16, 16, 10, 1)
    f = _field(16, 16)
    G.refresh(st, f, sad.RefreshMode.Full, 2, 4, 1, F32)
    st.bump()
    with pytest.raises(sad.StaleField):
        G.render_image(st, f, F32)
    f2 = _field(16, 16)
    f2.synced_generation = st.generation
    with pytest.raises(sad.EmptyList):
        G.render_image(st, f2, F32)
    with pytest.raises(sad.EmptyList):
        G.backward_image(st, f2, random_target(16, 16, 1), sad.GradBuffer(), F32)


# ---------------------------------------------------------------------------- optimiser / budget
def test_adam_bitwise(G, R):
    w, h = 40, 32
    st = random_model(w, h, 60, 3)
    st.frozen[7] = 1
    st.deactivate(9)
    rng = np.random.default_rng(3)
    g = sad.GradBuffer(st.size())
    g.data[:] = rng.normal(size=g.data.shape) * 1e-3
    g.data[5, 0] = np.nan
    a, b = st.copy(), st.copy()
    ma, mb = sad.AdamState(st.size()), sad.AdamState(st.size())
    cfg = sad.TrainConfig()
    for _ in range(3):
        G.adam_step(a, g, ma, w, h, cfg)
        R.adam_step(b, g, mb, w, h, cfg)
    for p in ("x", "y", "log_tau", "radius", "col_r", "col_g", "col_b", "dir_x", "dir_y", "aniso"):
        assert np.array_equal(getattr(a, p), getattr(b, p)), p
    assert np.array_equal(ma.m, mb.m) and np.array_equal(ma.v, mb.v)
    assert ma.t == mb.t == 3 and ma.skipped == mb.skipped


def test_stats_prune_densify(G, R):
    w, h = 48, 48
    st = random_model(w, h, 40, 11)
    tgt = random_target(w, h, 12)
    f = _field(w, h)
    R.refresh(st, f, sad.RefreshMode.Full, 4, 4, 7, F64)
    sg = G.accumulate_stats(st, f, tgt)
    sr = R.accumulate_stats(st, f, tgt)
    assert sg.valid_pixels == sr.valid_pixels
    assert np.array_equal(sg.data, sr.data)
    cfg = sad.TrainConfig()
    a, b = st.copy(), st.copy()
    assert G.prune(a, sr, 0.2) == R.prune(b, sr, 0.2)
    assert np.array_equal(a.active, b.active) and np.array_equal(a.x, b.x)
    ma, mb = sad.AdamState(a.size()), sad.AdamState(b.size())
    ma.m[:] = 0.5
    mb.m[:] = 0.5
    assert G.densify(a, ma, sr, tgt, 0.5, cfg) == R.densify(b, mb, sr, tgt, 0.5, cfg)
    for p in ("x", "y", "log_tau", "radius", "col_r", "dir_x", "dir_y", "aniso", "active"):
        assert np.array_equal(getattr(a, p), getattr(b, p)), p
    assert np.array_equal(ma.m, mb.m)


def test_densify_appends_and_cap(G, R):
    w, h = 48, 48
    st = random_model(w, h, 40, 21)
    tgt = random_target(w, h, 22)
    f = _field(w, h)
    R.refresh(st, f, sad.RefreshMode.Full, 4, 4, 7, F64)
    sr = R.accumulate_stats(st, f, tgt)
    for max_sites in (0, 45):
        cfg = sad.TrainConfig(max_sites=max_sites)
        a, b = st.copy(), st.copy()
        ma, mb = sad.AdamState(a.size()), sad.AdamState(b.size())
        dg = G.densify(a, ma, sr, tgt, 0.9, cfg)
        dr = R.densify(b, mb, sr, tgt, 0.9, cfg)
        assert dg == dr and a.size() == b.size()
        assert np.array_equal(a.x, b.x) and np.array_equal(a.active, b.active)


def test_init_sites_identical(G, R):
    for w, h, n in ((40, 32, 50), (256, 192, 3000)):
        tgt = synth_target(w, h, 5)
        a, b = sad.SiteStore(), sad.SiteStore()
        G.init_sites(a, tgt, n, sad.TrainConfig(seed=3))
        R.init_sites(b, tgt, n, sad.TrainConfig(seed=3))
        for p in ("x", "y", "col_r", "col_g", "col_b", "radius", "log_tau"):
            assert np.array_equal(getattr(a, p), getattr(b, p)), p


# ---------------------------------------------------------------------------- resident fit
def test_fit_small_budget_history(G, R):
    tgt = synth_target(32, 24, 2)
    cfg = sad.TrainConfig(iters=60, target_bpp=4.0, fp64=False, seed=5, densify_start=10, densify_every=10,
                          prune_start=20, prune_every=20)
    a = G.fit(tgt, cfg)
    b = R.fit(tgt, cfg)
    assert a.schedule_scale == b.schedule_scale
    ha = [r.psnr for r in a.history]
    hb = [r.psnr for r in b.history]
    assert np.max(np.abs(np.array(ha[:20]) - np.array(hb[:20]))) <= 0.05
    assert [r.active_sites for r in a.history][:20] == [r.active_sites for r in b.history][:20]


def test_fit_config1_first_iterations(G, R):
    """Config 1 (256x256, 4096 sites): PSNR trajectory within 0.05 dB over iterations 1-20."""
    tgt = synth_target(256, 256, 1)
    cfg = sad.TrainConfig(iters=20, n_sites=4096, fp64=False)
    a = G.fit(tgt, cfg)
    b = R.fit(tgt, cfg)
    d = np.abs(np.array([r.psnr for r in a.history]) - np.array([r.psnr for r in b.history]))
    assert d.max() <= 0.05, d


def test_fit_fp64_default_config(G, R):
    """The reference's TrainConfig defaults to fp64 (types.hpp:162): the all-double GPU fit is
    bit-identical too (device glibc-exp port; host glibc log for the split anisotropy)."""
    tgt = synth_target(32, 24, 6)
    cfg = sad.TrainConfig(iters=60, n_sites=60, seed=3)
    assert cfg.fp64
    a = G.fit(tgt, cfg)
    b = R.fit(tgt, cfg)
    assert [sad.history_line(r) for r in a.history] == [sad.history_line(r) for r in b.history]
    assert np.array_equal(a.sites.x, b.sites.x) and np.array_equal(a.field.ids, b.field.ids)
    # with the budget schedule (densify / prune events) as well
    cfg = sad.TrainConfig(iters=200, target_bpp=2.0, seed=3)
    a = G.fit(synth_target(64, 48, 2), cfg)
    b = R.fit(synth_target(64, 48, 2), cfg)
    assert [sad.history_line(r) for r in a.history] == [sad.history_line(r) for r in b.history]


def test_fit_deterministic(G):
    tgt = ramp_image(32, 32)
    cfg = sad.TrainConfig(iters=40, n_sites=25, seed=11, fp64=False)
    a = G.fit(tgt, cfg)
    b = G.fit(tgt, cfg)
    assert [sad.history_line(r) for r in a.history] == [sad.history_line(r) for r in b.history]
    assert np.array_equal(a.sites.x, b.sites.x) and np.array_equal(a.field.ids, b.field.ids)


def test_fit_frozen_survive(G):
    """test_train.cpp:427-457."""
    tgt = ramp_image(32, 32)
    cfg = sad.TrainConfig(iters=50, n_sites=16, seed=7, fp64=False)
    st = sad.SiteStore()
    G.init_sites(st, tgt, 16, cfg)
    p = st.get(3)
    p.x, p.y, p.log_tau, p.color, p.frozen = 5.123456789, 17.987654321, 8.25, (0.123456789, 0.5, 0.5), True
    st.set(3, p)
    st.frozen[8] = 1
    other = st.get(8)
    r = G.fit_store(st, tgt, cfg)
    q = r.sites.get(3)
    assert (q.x, q.y, q.log_tau, q.color[0]) == (5.123456789, 17.987654321, 8.25, 0.123456789)
    assert r.sites.get(8).x == other.x
