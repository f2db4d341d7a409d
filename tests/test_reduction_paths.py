"""GPU parity of the tile-reduction paths the reference's own tests force (test_grad.cpp:176-279), of the
record-pool fallbacks, of non-finite adjoints, and of the two entry points with no other test
(`exact_topk_batch`, candidates.cpp:198-248; `clamp_project`, train.cpp:113-137).

fp32 (and stats): the device groups each tile's per-(site, channel) contributions in a shared-memory
hash of UMAX = entries/4 local sites (sad_kernels.cu TileRed); beyond that, and when the per-site record
slots or the overflow-record pool run out, sums merge exactly into per-site double-double totals with
128-bit CAS.  fp64 gradients replay the reference's TileReducer itself (k_backward_ord: 16x16 tiles,
256 slots, 8 probes; an overflowed site's contributions become raw records), so the 320-site and
hash-collision cases below drive the reference's own overflow path on the device.  Every result must
equal the reference's bit for bit.
"""
import ctypes as C
import os

import numpy as np
import pytest

import paper_2604_21984_b200 as sad
from oracle.bindings import c_backend, have_ref, ref_backend
from paper_2604_21984_b200 import api
from tests.fixtures import random_model, random_target, synth_target

pytestmark = pytest.mark.gpu

F32 = sad.RunOpts(fp64=False)
F64 = sad.RunOpts(fp64=True)


@pytest.fixture(scope="module")
def G():
    return sad.gpu_backend(0)


@pytest.fixture(scope="module")
def R():
    return ref_backend() if have_ref() else c_backend()


def _synced_field(st, w, h, lists):
    f = sad.CandidateField()
    f.resize(w, h, 8)
    f.ids = np.ascontiguousarray(lists.reshape(-1).astype(np.uint32))
    f.synced_generation = st.generation
    return f


def _assert_backward_equal(G, R, st, f, tgt, opts, removal=True):
    gg, gr = sad.GradBuffer(), sad.GradBuffer()
    lg = G.backward_image(st, f, tgt, gg, opts, removal)
    lr = R.backward_image(st, f, tgt, gr, opts, removal)
    assert lg == lr
    assert np.array_equal(gg.data, gr.data)
    assert gg.nonfinite == gr.nonfinite
    return gg


def _assert_stats_equal(G, R, st, f, tgt):
    sg = G.accumulate_stats(st, f, tgt)
    sr = R.accumulate_stats(st, f, tgt)
    assert sg.valid_pixels == sr.valid_pixels
    assert np.array_equal(sg.data, sr.data)


@pytest.mark.parametrize("fp64", [False, True])
def test_tile_overflow_320_sites(G, R, fp64):
    """test_grad.cpp:176-232: lists (p*8+j) % 320 put 320 distinct sites into every tile — more than
    the device's UMAX (256 for the 16x8 fp32 tile, 128 for the 8x8 fp64 and stats tiles), so the
    hash table fills and entries take the exact DD-CAS path; the sums must stay exact."""
    w, h, n = 64, 64, 320
    st = random_model(w, h, n, 37)
    tgt = random_target(w, h, 38)
    p = np.arange(w * h)[:, None]
    lists = (p * 8 + np.arange(8)[None, :]) % n
    f = _synced_field(st, w, h, lists)
    _assert_backward_equal(G, R, st, f, tgt, sad.RunOpts(fp64=fp64), removal=True)
    _assert_backward_equal(G, R, st, f, tgt, sad.RunOpts(fp64=fp64), removal=False)
    if fp64:
        _assert_stats_equal(G, R, st, f, tgt)


def _device_hash_bucket_ids(count, bucket=1, stride=256):
    """Ids whose device tile hash ((id * 2654435761) & (HT - 1), HT = 256 or 128) collides: the low
    byte of the product depends only on id mod 256 (the multiplier is odd)."""
    return [bucket + stride * i for i in range(count)]


def _ref_hash_bucket_ids(count, want=None):
    """Ids sharing the reference's tile_hash bucket ((id * 2654435761) >> 24, grad.hpp:90)."""
    out = []
    h0 = None
    for i in range(1, 1 << 20):
        hv = ((i * 2654435761) & 0xFFFFFFFF) >> 24
        if h0 is None:
            h0 = hv
        if hv == h0:
            out.append(i)
            if len(out) == count:
                return out
    raise AssertionError


@pytest.mark.parametrize("fp64", [False, True])
def test_tile_hash_collisions(G, R, fp64):
    """test_grad.cpp:234-279: ten ids sharing one hash bucket, repeated across the tile — on the device
    hash (linear probing through a chain of ten) in the top half of the image, on the reference's
    hash (more keys than its 8 probes) in the bottom half."""
    dev = _device_hash_bucket_ids(10)
    ref = _ref_hash_bucket_ids(10)
    n = max(max(dev), max(ref)) + 1
    w, h = 48, 32
    st = random_model(w, h, n, 77)
    tgt = random_target(w, h, 78)
    p = np.arange(w * h)
    j = np.arange(8)[None, :]
    lists = np.where((p // w < h // 2)[:, None], np.array(dev)[(p[:, None] * 8 + j) % 10],
                     np.array(ref)[(p[:, None] * 3 + j) % 10])
    f = _synced_field(st, w, h, lists)
    _assert_backward_equal(G, R, st, f, tgt, sad.RunOpts(fp64=fp64), removal=True)
    _assert_stats_equal(G, R, st, f, tgt)


def _fresh_backend(env):
    """A second device context created under `env` (record-pool knobs are read at context creation)."""
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        lib = api.load_library()
        ctx = C.c_void_p()
        assert lib.sad_ctx_create(C.c_int(0), None, C.byref(ctx)) == 0
        return api.Backend(lib, "sad_", ctx=ctx)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def test_record_pool_exhaustion_per_call(R):
    """One record slot per (site, pass) (SAD_MAXT=1) and an 8-record overflow pool (SAD_OCAP=8):
    nearly every (site, tile) record takes the overflow list and then the exhausted-pool DD-CAS path;
    backward and stats must still equal the reference."""
    B = _fresh_backend({"SAD_MAXT": "1", "SAD_OCAP": "8"})
    try:
        w, h = 96, 80
        st = random_model(w, h, 150, 5)
        tgt = random_target(w, h, 6)
        f = sad.CandidateField()
        f.resize(w, h, 8)
        R.refresh(st, f, sad.RefreshMode.Full, 4, 4, 3, F32)
        for opts in (F32, F64):
            _assert_backward_equal(B, R, st, f, tgt, opts, removal=True)
        _assert_stats_equal(B, R, st, f, tgt)
    finally:
        B.lib.sad_ctx_destroy(B.ctx)


def test_record_pool_exhaustion_fit(R):
    """The resident fit with its adaptive record pool capped (SAD_APSIZE) and an 8-record overflow pool:
    every history line, the final sites and the map stay identical to the reference's fit."""
    B = _fresh_backend({"SAD_APSIZE": "64", "SAD_OCAP": "8"})
    try:
        tgt = synth_target(64, 48, 3)
        cfg = sad.TrainConfig(iters=80, target_bpp=3.0, fp64=False, seed=2)
        a = B.fit(tgt, cfg)
        b = R.fit(tgt, cfg)
        assert [sad.history_line(r) for r in a.history] == [sad.history_line(r) for r in b.history]
        assert np.array_equal(a.sites.x, b.sites.x) and np.array_equal(a.field.ids, b.field.ids)
        B.close()
    finally:
        B.lib.sad_ctx_destroy(B.ctx)


def test_fp64_ordered_fit_overflow_lists(R):
    """fp64 fit with the adaptive record pool capped at 64 records (SAD_APSIZE) and a large overflow pool:
    nearly every tagged (site, tile) record travels through the per-site overflow lists, whose order the
    ordered merge restores from the tags; the fit must equal the reference's."""
    B = _fresh_backend({"SAD_APSIZE": "64", "SAD_OCAP": "200000"})
    try:
        tgt = synth_target(64, 48, 5)
        cfg = sad.TrainConfig(iters=60, target_bpp=3.0, fp64=True, seed=4)
        a = B.fit(tgt, cfg)
        b = R.fit(tgt, cfg)
        assert [sad.history_line(r) for r in a.history] == [sad.history_line(r) for r in b.history]
        assert np.array_equal(a.sites.x, b.sites.x) and np.array_equal(a.field.ids, b.field.ids)
        B.close()
    finally:
        B.lib.sad_ctx_destroy(B.ctx)


@pytest.mark.parametrize("mode", ["backward", "removal", "pixgrad"])
def test_nonfinite_adjoint(G, R, mode):
    """A target with an inf pixel (and one huge value) makes g non-finite at those pixels: the
    reference scrubs and counts every 0 * inf = NaN term, zero-weight candidates included
    (grad.cpp:232-237); the device must count the same."""
    w, h = 48, 40
    st = random_model(w, h, 30, 9)
    st.log_tau[:] = 12.0  # sharp softmax: many candidates underflow to w == 0
    st.bump()
    tgt = random_target(w, h, 10)
    f = sad.CandidateField()
    f.resize(w, h, 8)
    R.refresh(st, f, sad.RefreshMode.Full, 4, 4, 3, F32)
    tgt.data[3 * (5 * w + 7) + 1] = np.inf
    tgt.data[3 * (20 * w + 30) + 2] = 3e38
    if mode == "pixgrad":
        dl = random_target(w, h, 11)
        dl.data -= 0.5
        dl.data[3 * (12 * w + 3)] = np.inf
        dl.data[3 * (30 * w + 40) + 1] = -np.inf
        gg, gr = sad.GradBuffer(), sad.GradBuffer()
        G.backward_pixel_grad(st, f, dl, gg, F32)
        R.backward_pixel_grad(st, f, dl, gr, F32)
        assert gg.nonfinite == gr.nonfinite and gr.nonfinite > 0
        assert np.array_equal(gg.data[:, :10], gr.data[:, :10])
        return
    for opts in (F32, F64):
        g = _assert_backward_equal(G, R, st, f, tgt, opts, removal=(mode == "removal"))
        assert g.nonfinite > 0


def test_pixgrad_size_mismatch(G, R):
    """backward_pixel_grad with an adjoint of the wrong size raises (grad.cpp:383-384) before reading it."""
    st = random_model(32, 24, 20, 1)
    f = sad.CandidateField()
    f.resize(32, 24, 8)
    R.refresh(st, f, sad.RefreshMode.Full, 2, 4, 1, F32)
    for B in (G, R):
        with pytest.raises(sad.api.InvalidArgument):
            B.backward_pixel_grad(st, f, sad.ImageBuffer(16, 24), sad.GradBuffer(), F32)


@pytest.mark.parametrize("fp64", [False, True])
@pytest.mark.parametrize("k", [1, 8, 16])
def test_exact_topk_batch(G, R, fp64, k):
    """exact_topk_batch (candidates.cpp:198-248): brute-force top-K under the unpacked ScoreTable logit
    over the active sites, identical ids per query."""
    w, h = 96, 64
    st = random_model(w, h, 700, 12)
    for i in range(0, 700, 9):
        st.deactivate(i)
    rng = np.random.default_rng(k)
    pix = np.stack([rng.integers(0, w, 500), rng.integers(0, h, 500)], 1)
    scale = sad.normalization_scale(w, h)
    a = G.exact_topk_batch(st, pix, k, scale, fp64)
    b = R.exact_topk_batch(st, pix, k, scale, fp64)
    assert np.array_equal(a, b)


def test_exact_topk_refresh_convergence(G, R):
    """The convergence check of test_candidates.cpp:196-222 with the GPU checker: after a full refresh the
    GPU map's lists agree with the GPU brute force on >= 95 % of probed cells, and the GPU brute force
    equals the reference's."""
    w, h = 128, 96
    st = random_model(w, h, 400, 3)
    f = sad.CandidateField()
    f.resize(w, h, 8)
    G.refresh(st, f, sad.RefreshMode.Full, 8, 4, 5, F32)
    rng = np.random.default_rng(0)
    pix = np.stack([rng.integers(0, w, 256), rng.integers(0, h, 256)], 1)
    scale = sad.normalization_scale(w, h)
    ex = G.exact_topk_batch(st, pix, 8, scale, False)
    assert np.array_equal(ex, R.exact_topk_batch(st, pix, 8, scale, False))
    ids = f.ids.reshape(h, w, 8)
    hit = sum(set(ids[y, x]) == set(ex[i]) for i, (x, y) in enumerate(pix))
    assert hit >= 0.95 * len(pix)


def test_clamp_project(G, R):
    """clamp_project (train.cpp:113-137) on out-of-range parameters, zero and non-finite directions, a
    NaN coordinate (std::min/std::max keep it), frozen and inactive sites (untouched)."""
    w, h = 40, 30
    st = random_model(w, h, 60, 8)
    rng = np.random.default_rng(8)
    st.x[:] = rng.uniform(-10, w + 10, st.size())
    st.y[:] = rng.uniform(-10, h + 10, st.size())
    st.log_tau[:] = rng.uniform(0, 25, st.size())
    st.radius[:] = rng.uniform(0, 600, st.size())
    st.aniso[:] = rng.uniform(-3, 3, st.size())
    st.col_r[:] = rng.uniform(-0.5, 1.5, st.size())
    st.col_g[:] = rng.uniform(-0.5, 1.5, st.size())
    st.col_b[:] = rng.uniform(-0.5, 1.5, st.size())
    st.dir_x[:] = rng.normal(size=st.size()) * 3
    st.dir_y[:] = rng.normal(size=st.size()) * 3
    st.dir_x[4] = st.dir_y[4] = 0.0
    st.dir_x[5], st.dir_y[5] = 1e-13, 0.0
    st.dir_x[6] = np.inf
    st.x[10] = np.nan
    st.frozen[11] = 1
    st.deactivate(12)
    st.bump()
    for clamp_color in (True, False):
        cfg = sad.TrainConfig(clamp_color=clamp_color)
        a, b = st.copy(), st.copy()
        G.clamp_project(a, w, h, cfg)
        R.clamp_project(b, w, h, cfg)
        for p in ("x", "y", "log_tau", "radius", "col_r", "col_g", "col_b", "dir_x", "dir_y", "aniso"):
            assert np.array_equal(getattr(a, p).view(np.uint64), getattr(b, p).view(np.uint64)), p
        assert a.generation == b.generation
