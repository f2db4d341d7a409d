"""Device-resident SiteStore / CandidateField (sad_sites_{alloc,upload,download},
sad_field_{alloc,upload,download}): a refresh -> render -> backward -> Adam -> event chain run on the
context's resident objects (NULL views across the C ABI, no host copies in between) gives bit-for-bit
the results of the host-view calls, with the reference's generation / pass-index bookkeeping."""
import numpy as np
import pytest

import paper_2604_21984_b200 as sad
from tests.fixtures import random_model, random_target

pytestmark = pytest.mark.gpu
F32 = sad.RunOpts(fp64=False)


def _field(w, h, k=8):
    f = sad.CandidateField()
    f.resize(w, h, k)
    return f


def test_resident_chain_matches_host_views():
    G = sad.gpu_backend(0)
    w, h = 64, 48
    st = random_model(w, h, 90, 7)
    tgt = random_target(w, h, 8)
    cfg = sad.TrainConfig()
    # host-view path
    f = _field(w, h)
    G.refresh(st, f, sad.RefreshMode.Full, 4, 4, 7, F32)
    G.refresh(st, f, sad.RefreshMode.WarmStart, 2, 4, 9, F32)
    img = G.render_image(st, f, F32).data
    g_host = sad.GradBuffer()
    l_host = G.backward_image(st, f, tgt, g_host, F32, False)
    st_host = st.copy()
    a_host = sad.AdamState(st.size())
    G.adam_step(st_host, g_host, a_host, w, h, cfg)

    # resident path
    S = G.sites_upload(st)
    F = G.field_alloc(w, h, 8)
    assert S.size() == st.size() and S.generation == st.generation
    G.refresh(S, F, sad.RefreshMode.Full, 4, 4, 7, F32)
    G.refresh(S, F, sad.RefreshMode.WarmStart, 2, 4, 9, F32)
    fd = G.field_download()
    assert np.array_equal(fd.ids, f.ids)
    assert (fd.pass_index, fd.refresh_count, fd.synced_generation) == (f.pass_index, f.refresh_count,
                                                                        f.synced_generation)
    assert np.array_equal(G.render_image(S, F, F32).data, img)
    g_res = sad.GradBuffer()
    assert G.backward_image(S, F, tgt, g_res, F32, False) == l_host
    assert np.array_equal(g_res.data, g_host.data)
    a_res = sad.AdamState(st.size())
    G.adam_step(S, g_res, a_res, w, h, cfg)
    sd = G.sites_download()
    for p in ("x", "y", "log_tau", "radius", "col_r", "dir_x", "dir_y", "aniso", "active"):
        assert np.array_equal(getattr(sd, p), getattr(st_host, p)), p
    assert sd.generation == st_host.generation
    assert np.array_equal(a_res.m, a_host.m) and a_res.t == a_host.t
    # sites moved: the resident field is stale for them, exactly like the reference's check_synced
    with pytest.raises(sad.StaleField):
        G.render_image(S, F, F32)


def test_resident_events_and_invalidation():
    G = sad.gpu_backend(0)
    w, h = 48, 48
    st = random_model(w, h, 40, 11)
    tgt = random_target(w, h, 12)
    cfg = sad.TrainConfig()
    f = _field(w, h)
    G.refresh(st, f, sad.RefreshMode.Full, 4, 4, 7, F32)
    stats = G.accumulate_stats(st, f, tgt)
    a, ma = st.copy(), sad.AdamState(st.size())
    G.prune(a, stats, 0.2)
    G.densify(a, ma, stats, tgt, 0.5, cfg)

    S = G.sites_upload(st)
    F = G.field_upload(f)
    rs = G.accumulate_stats(S, F, tgt)
    assert rs.valid_pixels == stats.valid_pixels and np.array_equal(rs.data, stats.data)
    mb = sad.AdamState(st.size())
    G.prune(S, rs, 0.2)
    # densify appends: re-upload the pruned store with room for the children
    cur = G.sites_download()
    S = G.sites_upload(cur, capacity=2 * cur.size())
    nd = G.densify(S, mb, rs, tgt, 0.5, cfg)
    sd = G.sites_download()
    assert nd > 0 and sd.size() == a.size()
    for p in ("x", "y", "log_tau", "radius", "active"):
        assert np.array_equal(getattr(sd, p), getattr(a, p)), p
    # a host-view call replaces the workspace copy: the resident sites are gone
    G.render_image(st, f, F32)
    with pytest.raises(sad.InvalidArgument):
        G.render_image(S, F, F32)


def test_oneshot_fit_and_fit_store():
    """sad_fit / sad_fit_store (one C call, what a cgo/JNI binding uses) equal the run-based API."""
    from tests.fixtures import synth_target
    G = sad.gpu_backend(0)
    tgt = synth_target(40, 32, 5)
    cfg = sad.TrainConfig(iters=60, target_bpp=4.0, fp64=False, seed=5, densify_start=10, densify_every=10,
                          prune_start=20, prune_every=20)
    a = G.fit(tgt, cfg)
    b = G.fit_oneshot(tgt, cfg)
    assert [sad.history_line(r) for r in a.history] == [sad.history_line(r) for r in b.history]
    assert a.schedule_scale == b.schedule_scale
    assert np.array_equal(a.field.ids, b.field.ids) and a.field.pass_index == b.field.pass_index
    for p in ("x", "y", "log_tau", "active"):
        assert np.array_equal(getattr(a.sites, p), getattr(b.sites, p)), p
    init = a.sites
    c = G.fit_store(init, tgt, sad.TrainConfig(iters=20, fp64=False, seed=2))
    d = G.fit_oneshot(tgt, sad.TrainConfig(iters=20, fp64=False, seed=2), init=init)
    assert [sad.history_line(r) for r in c.history] == [sad.history_line(r) for r in d.history]
    assert np.array_equal(c.sites.x, d.sites.x)
    # an undersized output store is refused
    import ctypes as C
    st = sad.SiteStore(0)
    sv, keep = st._view(capacity=1)
    cc = cfg.to_c()
    with pytest.raises(sad.api.CapacityError):
        G._call("fit", tgt.data.ctypes.data_as(C.POINTER(C.c_double)), C.c_int(40), C.c_int(32), C.byref(cc),
                C.byref(sv), None, None, None)


def test_cached_run_graphs_follow_buffer_reallocation():
    """A cached fit run replays CUDA graphs of plain iterations that hold raw buffer addresses: growing
    the run's capacity (a larger initial store) must drop them, and fits before and after the growth
    equal fresh one-shot fits."""
    from tests.fixtures import synth_target
    G = sad.gpu_backend(0)
    tgt = synth_target(48, 40, 7)
    cfg = sad.TrainConfig(iters=40, n_sites=60, fp64=False, seed=3)  # budget off: all iterations graph-replayed
    a = G.fit(tgt, cfg)
    big = G.fit(tgt, sad.TrainConfig(iters=5, n_sites=300, fp64=False, seed=4)).sites
    c = G.fit_store(big, tgt, cfg)  # same cached run, capacity 60 -> 300
    d = G.fit_oneshot(tgt, cfg, init=big)
    assert [sad.history_line(r) for r in c.history] == [sad.history_line(r) for r in d.history]
    for p in ("x", "y", "log_tau", "radius", "active"):
        assert np.array_equal(getattr(c.sites, p), getattr(d.sites, p)), p
    assert np.array_equal(c.field.ids, d.field.ids)
    e = G.fit(tgt, cfg)  # the grown run again from init_sites
    assert [sad.history_line(r) for r in e.history] == [sad.history_line(r) for r in a.history]
    assert np.array_equal(e.field.ids, a.field.ids)
