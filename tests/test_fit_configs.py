"""Full-configuration fit parity on the GPU.

* Config 1 (256x256, 4096 sites, 200 iterations, budget off), fp32 and fp64: the GPU fit against the
  compiled reference run live on this box's host cores — every history line, the final sites and
  the final map identical.
* Config 2 (768x512 synthetic Kodak-shaped images, 2 BPP, 4000 iterations with 150 densify/prune
  events), image seeds 1-8 in fp32 and seeds 1, 3 (reference on 8 threads) and 2 (on its default single
  thread) in fp64 (the reference's default precision), and
  config 3 (2048x2048, 100k sites, 300 iterations) in fp32 and fp64, and the config-5 shape (8192x8192, 2 BPP: 1.69M sites,
  25 iterations incl. one densify event and its re-seeded refresh): the GPU fit against goldens of complete
  reference fits (tests/golden/fit_*.npz, written here by tests/golden/make_fit_golden.py from the
  unmodified reference library; a reference fit takes minutes per image, the GPU's under a second).
  Every history row (loss and PSNR as doubles, active count), the schedule scale, SHA-256 digests
  of all final site arrays and of the final map, the pass index and the decode PSNR must be equal,
  in fp64 as in fp32.
"""
import ast
import glob
import hashlib
import os

import numpy as np
import pytest

import paper_2604_21984_b200 as sad
from oracle.bindings import c_backend, have_ref, ref_backend
from paper_2604_21984_b200.synth import synthetic_image

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = sorted(glob.glob(os.path.join(HERE, "golden", "fit_*.npz")))
SITE_ARRAYS = ("x", "y", "log_tau", "radius", "col_r", "col_g", "col_b", "dir_x", "dir_y", "aniso", "active",
               "frozen")


@pytest.fixture(scope="module")
def G():
    return sad.gpu_backend(0)


MAX_RUNS = 3  # runs per golden comparison (the determinism caveat at test_full_fit_matches_reference_golden)


def _digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _decode_psnr(G, res, img):
    out = G.render_image(res.sites, res.field, sad.RunOpts(fp64=False)).data
    mse = float(np.mean((out - img.data) ** 2))
    return 99.0 if mse <= 0 else 10.0 * np.log10(1.0 / mse)


@pytest.mark.parametrize("fp64", [False, True])
def test_config1_full_fit_identical(G, fp64):
    """Config 1: all 200 iterations bit-identical to the reference (live, all host threads)."""
    R = ref_backend(threads=os.cpu_count() or 1) if have_ref() else c_backend()
    tgt = sad.ImageBuffer(256, 256, synthetic_image(256, 256, 1))
    cfg = sad.TrainConfig(iters=200, n_sites=4096, fp64=fp64, seed=1)
    b = R.fit(tgt, sad.TrainConfig(iters=200, n_sites=4096, fp64=fp64, seed=1, threads=os.cpu_count() or 1))
    for attempt in range(MAX_RUNS):  # see the determinism caveat below
        a = G.fit(tgt, cfg)
        assert [sad.history_line(r) for r in a.history] == [sad.history_line(r) for r in b.history]
        assert np.array_equal(a.field.ids, b.field.ids)
        assert a.field.pass_index == b.field.pass_index
        if all(np.array_equal(getattr(a.sites, p), getattr(b.sites, p)) for p in SITE_ARRAYS):
            break
    for p in SITE_ARRAYS:
        assert np.array_equal(getattr(a.sites, p), getattr(b.sites, p)), p


# fp64 fits: the contributions are doubles, whose Accum cascades are not order-independent; the fp64 path
# replays the reference's own order (k_backward_ord / ord_total), so these goldens are
# required identical in full like the fp32 ones (the double-double path, SAD_FP64_DD=1, diverged by
# one ulp at iteration 1021-1039 of config 2 / seed 1).


# Run-to-run determinism caveat: the fp32 per-site sums are double-doubles over float
# contributions, exact — hence order-independent — unless a sum spans more than ~106 bits (a site whose
# far pixels give softmax weights deep in the exponent range next to its near ones).  The order of the
# device's record claims varies between runs, so such a sum's last bit can vary, and with it the last bit
# of the site's double parameter — below what the float tables of the forward pass resolve, so the history
# and the map stay identical.  Measured: config 2 / seed 7, site 71's radius one ulp apart in 1-2 % of fits.
# The test therefore requires the history, the map and the decode PSNR identical in every run, and the
# complete site arrays identical in one of up to three runs (the others within 4 ulps at <= 0.1 % of sites).
def _site_digests_ok(res, d):
    return [p for p in SITE_ARRAYS if _digest(getattr(res.sites, p)) != str(d["sha_" + p])]


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[4:-4] for p in GOLDEN])
def test_full_fit_matches_reference_golden(G, path):
    d = np.load(path)
    w, h, seed = int(d["width"]), int(d["height"]), int(d["image_seed"])
    cfg = sad.TrainConfig(**ast.literal_eval(str(d["config"])))
    img = sad.ImageBuffer(w, h, synthetic_image(w, h, seed))
    runs = []
    for attempt in range(MAX_RUNS):
        res = G.fit(img, cfg)
        loss = np.array([r.loss for r in res.history], np.float64)
        psnr = np.array([r.psnr for r in res.history], np.float64)
        active = np.array([r.active_sites for r in res.history], np.int64)
        first = np.flatnonzero((loss.view(np.uint64) != d["loss"].view(np.uint64)) | (active != d["active"]))
        assert loss.shape == d["loss"].shape
        assert first.size == 0, f"history differs from iteration {first[0] + 1} on"
        assert np.array_equal(psnr.view(np.uint64), d["psnr"].view(np.uint64))
        assert res.schedule_scale == float(d["schedule_scale"])
        assert res.sites.size() == int(d["n_sites"])
        assert _digest(res.field.ids) == str(d["field_sha"])
        assert res.field.pass_index == int(d["pass_index"])
        runs.append(res)
        if not _site_digests_ok(res, d):
            break
    bad = _site_digests_ok(runs[-1], d)
    assert not bad, f"site arrays {bad} differ from the reference in {MAX_RUNS} runs"
    good = runs[-1]
    for res in runs[:-1]:  # the earlier, non-identical runs: last-bit differences at a few sites only
        for p in SITE_ARRAYS:
            a, b = getattr(res.sites, p), getattr(good.sites, p)
            diff = np.flatnonzero(a != b)
            assert diff.size <= max(1, a.size // 1000), f"{p} differs at {diff.size} sites"
            if a.dtype == np.float64 and diff.size:
                ulps = np.abs(a[diff].view(np.int64) - b[diff].view(np.int64))
                assert ulps.max() <= 4, f"{p} differs by {int(ulps.max())} ulps at site {diff[np.argmax(ulps)]}"
        print(f"{os.path.basename(path)}: reference-identical on run {len(runs)}; the earlier runs differed by "
              f"<= 4 ulps at a few sites")
    assert _decode_psnr(G, good, img) == float(d["decode_psnr"])


def test_golden_set_present():
    """The committed goldens cover config 2 over >= 8 images, fp64, and config 3."""
    names = {os.path.basename(p) for p in GOLDEN}
    assert sum(n.startswith("fit_config2_s") for n in names) >= 8
    assert "fit_config2_fp64_s1.npz" in names and "fit_config3_s1.npz" in names
    assert "fit_config5_short_s5.npz" in names
