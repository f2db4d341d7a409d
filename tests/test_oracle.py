"""CPU tests (no GPU): pin the plain-C restatement oracle (oracle/_ref/libsado.so) against the
compiled reference library (oracle/_ref/libsadref.so) and the committed golden vectors.

The restatement is what the GPU parity tests fall back to when the reference library is absent, so
it has to reproduce the reference bit for bit on the same inputs.
"""
import numpy as np
import pytest

import paper_2604_21984_b200 as sad
from oracle.bindings import c_backend, have_ref, ref_backend
from tests.fixtures import random_model, random_sites, random_target, ramp_image, synth_target

needs_ref = pytest.mark.skipif(not have_ref(), reason="reference library not built (no /root/reference)")


@pytest.fixture(scope="module")
def R():
    return ref_backend()


@pytest.fixture(scope="module")
def O():
    return c_backend()


F32 = sad.RunOpts(fp64=False)
F64 = sad.RunOpts(fp64=True)


@needs_ref
def test_rng_and_half_match(R, O):
    rng = np.random.default_rng(0)
    for s, a, b in rng.integers(0, 2**32, size=(200, 3), dtype=np.uint64):
        s = int(s) | (int(s) << 17)
        assert O.lib.sado_seeded_state(s, int(a), int(b)) == R.lib.sadref_seeded_state(s, int(a), int(b))
    bits = np.concatenate([rng.integers(0, 2**32, 20000, dtype=np.uint64).astype(np.uint32),
                           np.array([0, 0x80000000, 0x7f800000, 0xff800000, 0x33800000, 0x387fc000, 0x477fe000,
                                     0x477ff000, 0x38800000, 0x33000001], np.uint32)])
    f = bits.view(np.float32)
    for x in f:
        if np.isnan(x):
            continue
        hr = R.lib.sadref_float_to_half(float(x))
        assert O.lib.sado_float_to_half(float(x)) == hr
    for hb in range(0, 65536, 7):
        a, b = R.lib.sadref_half_to_float(hb), O.lib.sado_half_to_float(hb)
        assert (a == b) or (np.isnan(a) and np.isnan(b))


@needs_ref
def test_schedule_helpers(R, O):
    for b in (2, 4, 1024, 2048):
        for t in range(14):
            assert R.jump_step(t, b) == O.jump_step(t, b)
    for gw, gh in ((768, 512), (1, 1), (33, 7), (2048, 2048)):
        assert R.full_refresh_passes(gw, gh, 4) == O.full_refresh_passes(gw, gh, 4)
    cfg = sad.TrainConfig()
    for n0 in (100, 9831, 20000):
        for sc in (0.0, 0.3, 0.95):
            assert R.simulate_schedule(n0, sc, cfg) == O.simulate_schedule(n0, sc, cfg)
        assert R.plan_schedule(n0, 6144, cfg) == O.plan_schedule(n0, 6144, cfg)
    assert R.bpp_target_count(2.0, 768, 512) == O.bpp_target_count(2.0, 768, 512) == 6144


@needs_ref
@pytest.mark.parametrize("fp64", [False, True])
def test_refresh_maps_identical(R, O, fp64):
    opts = sad.RunOpts(fp64=fp64)
    for (w, h, n, seed) in ((24, 16, 40, 99), (64, 48, 120, 5), (37, 29, 60, 8)):
        st = random_sites(w, h, n, seed)
        st.deactivate(3)
        fr, fo = sad.CandidateField(), sad.CandidateField()
        fr.resize(w, h, 8)
        fo.resize(w, h, 8)
        R.refresh(st, fr, sad.RefreshMode.Full, 4, 4, 1234, opts)
        O.refresh(st, fo, sad.RefreshMode.Full, 4, 4, 1234, opts)
        assert np.array_equal(fr.ids, fo.ids)
        assert fr.pass_index == fo.pass_index
        R.refresh(st, fr, sad.RefreshMode.WarmStart, 2, 4, 77, opts)
        O.refresh(st, fo, sad.RefreshMode.WarmStart, 2, 4, 77, opts)
        assert np.array_equal(fr.ids, fo.ids)


@needs_ref
def test_refresh_other_k_and_cell(R, O):
    st = random_model(40, 30, 70, 4)
    for k, cell in ((3, 1), (12, 1), (8, 3), (16, 2)):
        fr, fo = sad.CandidateField(), sad.CandidateField()
        fr.resize(40, 30, k, cell)
        fo.resize(40, 30, k, cell)
        R.refresh(st, fr, sad.RefreshMode.Full, 3, 5, 9, F32)
        O.refresh(st, fo, sad.RefreshMode.Full, 3, 5, 9, F32)
        assert np.array_equal(fr.ids, fo.ids), (k, cell)


@needs_ref
@pytest.mark.parametrize("fp64", [False, True])
def test_render_and_backward_bitwise(R, O, fp64):
    opts = sad.RunOpts(fp64=fp64)
    st = random_model(64, 48, 90, 7)
    tgt = random_target(64, 48, 8)
    f = sad.CandidateField()
    f.resize(64, 48, 8)
    R.refresh(st, f, sad.RefreshMode.Full, 4, 4, 7, opts)
    assert np.array_equal(R.render_image(st, f, opts).data, O.render_image(st, f, opts).data)
    for rem in (False, True):
        gr, go = sad.GradBuffer(), sad.GradBuffer()
        lr = R.backward_image(st, f, tgt, gr, opts, rem)
        lo = O.backward_image(st, f, tgt, go, opts, rem)
        assert lr == lo
        assert np.array_equal(gr.data, go.data)
        assert gr.nonfinite == go.nonfinite
    assert R.image_loss(st, f, tgt, opts) == O.image_loss(st, f, tgt, opts)
    assert np.array_equal(R.render_id_map(st, f), O.render_id_map(st, f))


@needs_ref
def test_stats_prune_densify_bitwise(R, O):
    w, h = 48, 48
    st = random_model(w, h, 40, 11)
    tgt = random_target(w, h, 12)
    f = sad.CandidateField()
    f.resize(w, h, 8)
    R.refresh(st, f, sad.RefreshMode.Full, 4, 4, 7, F64)
    sr = R.accumulate_stats(st, f, tgt)
    so = O.accumulate_stats(st, f, tgt)
    assert sr.valid_pixels == so.valid_pixels
    assert np.array_equal(sr.data, so.data)
    cfg = sad.TrainConfig()
    a, b = st.copy(), st.copy()
    assert R.prune(a, sr, 0.2) == O.prune(b, so, 0.2)
    assert np.array_equal(a.active, b.active) and np.array_equal(a.x, b.x)
    ar, ao = sad.AdamState(a.size()), sad.AdamState(b.size())
    ar.m[:] = 0.5
    ao.m[:] = 0.5
    dr = R.densify(a, ar, sr, tgt, 0.5, cfg)
    do = O.densify(b, ao, so, tgt, 0.5, cfg)
    assert dr == do and dr > 0
    for p in ("x", "y", "log_tau", "radius", "col_r", "dir_x", "dir_y", "aniso", "active"):
        assert np.array_equal(getattr(a, p), getattr(b, p)), p
    assert np.array_equal(ar.m, ao.m)


@needs_ref
def test_adam_and_init_bitwise(R, O):
    w, h = 40, 32
    tgt = ramp_image(w, h)
    cfg = sad.TrainConfig()
    a, b = sad.SiteStore(), sad.SiteStore()
    R.init_sites(a, tgt, 50, cfg)
    O.init_sites(b, tgt, 50, cfg)
    for p in ("x", "y", "col_r", "col_b", "radius"):
        assert np.array_equal(getattr(a, p), getattr(b, p)), p
    rng = np.random.default_rng(3)
    g = sad.GradBuffer(a.size())
    g.data[:] = rng.normal(size=g.data.shape) * 1e-3
    g.data[5, 0] = np.nan
    a.frozen[7] = b.frozen[7] = 1
    ma, mb = sad.AdamState(a.size()), sad.AdamState(b.size())
    for _ in range(3):
        R.adam_step(a, g, ma, w, h, cfg)
        O.adam_step(b, g, mb, w, h, cfg)
    for p in ("x", "y", "log_tau", "radius", "col_r", "dir_x", "dir_y", "aniso"):
        assert np.array_equal(getattr(a, p), getattr(b, p)), p
    assert np.array_equal(ma.v, mb.v) and ma.skipped == mb.skipped == 3 and ma.t == 3


@needs_ref
def test_fit_history_bitwise_small(R, O):
    tgt = synth_target(32, 24, 2)
    cfg = sad.TrainConfig(iters=60, target_bpp=4.0, fp64=False, seed=5, densify_start=10, densify_every=10,
                          prune_start=20, prune_every=20)
    a = R.fit(tgt, cfg)
    b = O.fit(tgt, cfg)
    assert [sad.history_line(r) for r in a.history] == [sad.history_line(r) for r in b.history]
    assert a.schedule_scale == b.schedule_scale
    assert np.array_equal(a.field.ids, b.field.ids)
    assert np.array_equal(a.sites.x, b.sites.x)


def test_c_oracle_standalone_invariants(O):
    """Runs without the reference: list invariants of the restated propagate (sentinel tail, distinct
    active ids, strict (logit desc, id asc) order under the half-packed score)."""
    w, h = 32, 24
    st = random_sites(w, h, 50, 3)
    st.deactivate(10)
    f = sad.CandidateField()
    f.resize(w, h, 8)
    O.refresh(st, f, sad.RefreshMode.Full, 4, 4, 3, F64)
    ids = f.ids.reshape(h, w, 8)
    for gy in range(h):
        for gx in range(w):
            lst = [int(i) for i in ids[gy, gx] if i != sad.types.EMPTY]
            k = len(lst)
            assert all(i == sad.types.EMPTY for i in ids[gy, gx][k:])
            assert len(set(lst)) == k and 10 not in lst
