"""Golden vectors (tests/golden/*.npz, generated from the compiled reference by make_golden.py):
the plain-C oracle must reproduce them exactly on the CPU, and the CUDA library on the GPU.  These
pin both checkers where the reference library itself is not available (e.g. the GPU box)."""
import os

import numpy as np
import pytest

import paper_2604_21984_b200 as sad
from oracle.bindings import c_backend
from paper_2604_21984_b200.synth import Rng

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
PARAMS = ("x", "y", "log_tau", "radius", "col_r", "col_g", "col_b", "dir_x", "dir_y", "aniso", "active", "frozen")


def load(name):
    return dict(np.load(os.path.join(GOLD, name)))


def store(d, prefix="s_"):
    st = sad.SiteStore(0)
    for p in PARAMS:
        setattr(st, p, d[prefix + p].copy())
    return st


def field(ids, w, h, k=8):
    f = sad.CandidateField()
    f.resize(w, h, k)
    f.ids = ids.astype(np.uint32).copy()
    return f


def same_sites(st, d, prefix):
    return all(np.array_equal(getattr(st, p), d[prefix + p]) for p in PARAMS)


def backends():
    out = [pytest.param("c", id="c_oracle")]
    out.append(pytest.param("gpu", id="cuda", marks=pytest.mark.gpu))
    return out


def get(kind):
    return c_backend() if kind == "c" else sad.gpu_backend(0)


def test_core_rng_half():
    d = load("core.npz")
    O = c_backend()
    for (s, a, b), st0, seq in zip(d["triples"], d["states"], d["seqs"]):
        assert O.lib.sado_seeded_state(int(s), int(a), int(b)) == st0
        r = Rng(int(s), int(a), int(b))
        assert r.s == st0 and [r.next() for _ in range(16)] == list(seq)
    for f, hb in zip(d["floats"], d["halves"]):
        assert O.lib.sado_float_to_half(float(f)) == hb


@pytest.mark.parametrize("kind", backends())
def test_golden_refresh(kind):
    B = get(kind)
    d = load("refresh.npz")
    st = store(d)
    for fp64 in (0, 1):
        f = sad.CandidateField()
        f.resize(24, 16, 8)
        B.refresh(st, f, sad.RefreshMode.Full, 4, 4, 1234, sad.RunOpts(fp64=bool(fp64)))
        assert np.array_equal(f.ids, d[f"full_{fp64}"])
        B.refresh(st, f, sad.RefreshMode.WarmStart, 2, 4, 77, sad.RunOpts(fp64=bool(fp64)))
        assert np.array_equal(f.ids, d[f"warm_{fp64}"]) and f.pass_index == d[f"pass_index_{fp64}"][0]


@pytest.mark.parametrize("kind", backends())
def test_golden_render_backward(kind):
    B = get(kind)
    d = load("render_grad.npz")
    st = store(d)
    f = field(d["ids"], 64, 48)
    f.synced_generation = st.generation
    tgt = sad.ImageBuffer(64, 48, d["target"])
    for fp64 in (0, 1):
        opts = sad.RunOpts(fp64=bool(fp64))
        img = B.render_image(st, f, opts).data
        ref = d[f"render_{fp64}"]
        assert np.all(np.abs(img - ref) <= 1e-5 * np.maximum(np.abs(ref), 1e-3))
        if not fp64:
            assert np.array_equal(img, ref)
        g = sad.GradBuffer()
        loss = B.backward_image(st, f, tgt, g, opts, True)
        assert abs(loss - d[f"loss_{fp64}"][0]) <= 1e-7 * abs(d[f"loss_{fp64}"][0])
        for k in range(11):
            rk = d[f"grads_{fp64}"][:, k]
            assert np.linalg.norm(g.data[:, k] - rk) <= 1e-5 * np.linalg.norm(rk)
        if not fp64:
            assert loss == d["loss_0"][0] and np.array_equal(g.data, d["grads_0"])
    assert np.array_equal(B.render_id_map(st, f), d["id_map"])


@pytest.mark.parametrize("kind", backends())
def test_golden_budget(kind):
    B = get(kind)
    d = load("budget.npz")
    st = store(d)
    f = field(d["ids"], 48, 48)
    f.synced_generation = st.generation
    tgt = sad.ImageBuffer(48, 48, d["target"])
    s = B.accumulate_stats(st, f, tgt)
    assert s.valid_pixels == d["valid"][0]
    # double exp on the device may differ from glibc by an ulp; removal sums can cancel, so the bound
    # is relative to each channel's scale
    scale = np.max(np.abs(d["stats"]), axis=0, keepdims=True)
    assert np.all(np.abs(s.data - d["stats"]) <= 1e-12 * np.abs(d["stats"]) + 1e-13 * scale)
    ref = sad.StatsResult(st.size())
    ref.data, ref.valid_pixels = d["stats"], int(d["valid"][0])
    a = st.copy()
    assert B.prune(a, ref, 0.2) == d["pruned"][0]
    adam = sad.AdamState(a.size())
    adam.m[:] = 0.5
    assert B.densify(a, adam, ref, tgt, 0.5, sad.TrainConfig()) == d["densified"][0]
    assert same_sites(a, d, "out_") and np.array_equal(adam.m, d["adam_m"])


@pytest.mark.parametrize("kind", backends())
def test_golden_init_adam(kind):
    B = get(kind)
    d = load("train.npz")
    from tests.fixtures import ramp_image
    st = sad.SiteStore()
    B.init_sites(st, ramp_image(40, 32), 50, sad.TrainConfig())
    assert same_sites(st, d, "init_")
    st.frozen[7] = 1
    g = sad.GradBuffer(st.size())
    g.data = d["grads"].copy()
    m = sad.AdamState(st.size())
    for _ in range(3):
        B.adam_step(st, g, m, 40, 32, sad.TrainConfig())
    assert same_sites(st, d, "adam_") and np.array_equal(m.m, d["m"]) and np.array_equal(m.v, d["v"])
    assert m.skipped == d["skipped"][0]


@pytest.mark.parametrize("kind", backends())
def test_golden_fit(kind):
    B = get(kind)
    d = load("fit.npz")
    cfg = sad.TrainConfig(iters=60, target_bpp=4.0, fp64=False, seed=5, densify_start=10, densify_every=10,
                          prune_start=20, prune_every=20)
    r = B.fit(sad.ImageBuffer(32, 24, d["target"]), cfg)
    assert r.schedule_scale == d["scale"][0]
    assert np.array_equal([h.loss for h in r.history], d["loss"])
    assert np.array_equal([h.active_sites for h in r.history], d["active"])
    assert np.array_equal(r.field.ids, d["ids"]) and same_sites(r.sites, d, "out_")
