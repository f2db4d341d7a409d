"""tau_diffusion (train.cpp:171-213): the optional logtau-gradient smoothing stage of the fit.

CPU tests pin the C restatement against the compiled reference and port the reference's own test
(test_train.cpp:322-370); GPU tests compare the CUDA path (owner map -> edge sort/unique -> per-owner
sequential sums) with the reference per call and inside a full fit (bit-exact history).
"""
import numpy as np
import pytest

import paper_2604_21984_b200 as sad
from oracle.bindings import c_backend, have_ref, ref_backend
from tests.fixtures import random_model, synth_target

needs_ref = pytest.mark.skipif(not have_ref(), reason="reference library not built")


@pytest.fixture(scope="module")
def O():
    return c_backend()


def _two_sites():
    """test_train.cpp:323-340: two sites on an 8x8 image, gradients logtau +2 / -2, x 5."""
    st = sad.SiteStore(0)
    st.append(sad.Site(x=2, y=4, log_tau=9.0, radius=2.0))
    st.append(sad.Site(x=6, y=4, log_tau=9.0, radius=2.0))
    return st


def _grads(n, vals):
    g = sad.GradBuffer(n)
    for (site, slot), v in vals.items():
        g.data[site, slot] = v
    return g


def _reference_case(B):
    st = _two_sites()
    f = sad.CandidateField()
    f.resize(8, 8, 8)
    B.refresh(st, f, sad.RefreshMode.Full, 4, 4, 7, sad.RunOpts())
    base = {(0, 2): 2.0, (1, 2): -2.0, (0, 0): 5.0}
    g = _grads(2, base)
    B.tau_diffusion(st, f, 0.0, g)
    assert g.grad(2, 0) == 2.0 and g.grad(2, 1) == -2.0
    g = _grads(2, base)
    B.tau_diffusion(st, f, 1.0, g)
    assert abs(g.grad(2, 0)) <= 1e-12 and abs(g.grad(2, 1)) <= 1e-12
    assert g.grad(0, 0) == 5.0  # other channels untouched
    g = _grads(2, base)
    B.tau_diffusion(st, f, 0.5, g)
    assert g.grad(2, 0) == pytest.approx(1.0, rel=1e-12) and g.grad(2, 1) == pytest.approx(-1.0, rel=1e-12)
    # a site owning no pixels keeps its gradient
    shadow = st.get(0)
    shadow.radius = 1.0
    st.append(shadow)
    B.refresh(st, f, sad.RefreshMode.Full, 4, 4, 7, sad.RunOpts())
    g3 = _grads(3, {(0, 2): 2.0, (1, 2): -2.0, (2, 2): 7.0})
    B.tau_diffusion(st, f, 1.0, g3)
    assert g3.grad(2, 2) == 7.0
    with pytest.raises(sad.InvalidArgument):
        B.tau_diffusion(st, f, 1.5, g3)


def _random_case(seed):
    w, h = 48, 40
    st = random_model(w, h, 70, seed)
    st.deactivate(5)
    rng = np.random.default_rng(seed)
    g = sad.GradBuffer(st.size())
    g.data[:] = rng.normal(size=g.data.shape)
    return w, h, st, g


def test_reference_case_c_oracle(O):
    _reference_case(O)


@needs_ref
def test_reference_case_reference():
    _reference_case(ref_backend())


@needs_ref
@pytest.mark.parametrize("lam", [0.25, 0.5, 1.0])
def test_c_oracle_matches_reference(O, lam):
    R = ref_backend()
    w, h, st, g = _random_case(4)
    f = sad.CandidateField()
    f.resize(w, h, 8)
    R.refresh(st, f, sad.RefreshMode.Full, 4, 4, 9, sad.RunOpts())
    a = sad.GradBuffer()
    a.data = g.data.copy()
    b = sad.GradBuffer()
    b.data = g.data.copy()
    R.tau_diffusion(st, f, lam, a)
    O.tau_diffusion(st, f, lam, b)
    assert np.array_equal(a.data.view(np.uint64), b.data.view(np.uint64))
    assert not np.array_equal(a.data[:, 2], g.data[:, 2])


@needs_ref
def test_fit_with_tau_c_oracle_matches_reference(O):
    R = ref_backend()
    tgt = synth_target(32, 24, 3)
    cfg = sad.TrainConfig(iters=40, target_bpp=4.0, fp64=False, seed=5, densify_start=10, densify_every=10,
                          prune_start=20, prune_every=20, tau_diffusion_lambda=0.3)
    a = R.fit(tgt, cfg)
    b = O.fit(tgt, cfg)
    assert [sad.history_line(r) for r in a.history] == [sad.history_line(r) for r in b.history]
    assert np.array_equal(a.sites.log_tau, b.sites.log_tau)


# ---------------------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_reference_case_gpu():
    _reference_case(sad.gpu_backend(0))


@pytest.mark.gpu
@pytest.mark.parametrize("lam", [0.25, 1.0])
@pytest.mark.parametrize("cell", [1, 2])
def test_gpu_matches_oracle(lam, cell):
    G = sad.gpu_backend(0)
    Rb = ref_backend() if have_ref() else c_backend()
    w, h, st, g = _random_case(11)
    f = sad.CandidateField()
    f.resize(w, h, 8, cell)
    Rb.refresh(st, f, sad.RefreshMode.Full, 4, 4, 9, sad.RunOpts())
    a = sad.GradBuffer()
    a.data = g.data.copy()
    b = sad.GradBuffer()
    b.data = g.data.copy()
    G.tau_diffusion(st, f, lam, a)
    Rb.tau_diffusion(st, f, lam, b)
    assert np.array_equal(a.data.view(np.uint64), b.data.view(np.uint64))


@pytest.mark.gpu
def test_gpu_fit_with_tau_bitwise():
    """The resident fit with lambda > 0 (site totals -> owner map -> edge sort/unique -> mix -> Adam on
    the mixed totals) reproduces the reference fit's history and final sites exactly."""
    G = sad.gpu_backend(0)
    Rb = ref_backend() if have_ref() else c_backend()
    tgt = synth_target(48, 32, 4)
    cfg = sad.TrainConfig(iters=80, target_bpp=4.0, fp64=False, seed=5, densify_start=10, densify_every=10,
                          prune_start=20, prune_every=20, tau_diffusion_lambda=0.3)
    a = G.fit(tgt, cfg)
    b = Rb.fit(tgt, cfg)
    assert [sad.history_line(r) for r in a.history] == [sad.history_line(r) for r in b.history]
    for p in ("x", "y", "log_tau", "radius", "col_r", "aniso", "active"):
        assert np.array_equal(getattr(a.sites, p), getattr(b.sites, p)), p
    assert np.array_equal(a.field.ids, b.field.ids)
    # and the stage matters: lambda = 0 gives a different trajectory
    c = G.fit(tgt, sad.TrainConfig(iters=80, target_bpp=4.0, fp64=False, seed=5, densify_start=10,
                                   densify_every=10, prune_start=20, prune_every=20))
    assert not np.array_equal(a.sites.log_tau[: c.sites.size()], c.sites.log_tau[: a.sites.size()])


@pytest.mark.gpu
def test_gpu_fit_lambda_out_of_range():
    G = sad.gpu_backend(0)
    tgt = synth_target(16, 16, 1)
    with pytest.raises(sad.InvalidArgument):
        G.fit(tgt, sad.TrainConfig(iters=2, n_sites=20, fp64=False, tau_diffusion_lambda=1.5))
