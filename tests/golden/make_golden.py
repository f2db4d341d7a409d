"""Generates tests/golden/*.npz from the compiled reference library (oracle/_ref/libsadref.so, built
from /root/reference/proj/src by oracle/Makefile).  Run here (the reference is not on the GPU box):

    python tests/golden/make_golden.py

Every case uses the seeded generators of tests/fixtures.py (ports of the reference tests' own
fixtures), stores its inputs and the reference outputs, and is checked by tests/test_golden.py
against the plain-C oracle (CPU) and the CUDA library (GPU).
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import numpy as np  # noqa: E402

import paper_2604_21984_b200 as sad  # noqa: E402
from oracle.bindings import ref_backend  # noqa: E402
from paper_2604_21984_b200.synth import Rng  # noqa: E402
from tests.fixtures import random_model, random_sites, random_target, ramp_image, synth_target  # noqa: E402

PARAMS = ("x", "y", "log_tau", "radius", "col_r", "col_g", "col_b", "dir_x", "dir_y", "aniso", "active", "frozen")


def sites_dict(st, prefix="s_"):
    return {prefix + p: getattr(st, p).copy() for p in PARAMS}


def main():
    R = ref_backend()
    out = {}
    F32, F64 = sad.RunOpts(fp64=False), sad.RunOpts(fp64=True)

    # core: rng streams and half conversion (rng.hpp, half.hpp)
    triples = np.array([[1, 2, 3], [0xDEADBEEF, 0x1717, 0], [99, 0, 0], [5, 7, 9], [2**40 + 3, 1, 1]], np.uint64)
    states = [R.lib.sadref_seeded_state(int(s), int(a), int(b)) for s, a, b in triples]
    seqs = []
    for st0 in states:
        r = Rng(0, 0, 0)
        r.s = st0
        seqs.append([r.next() for _ in range(16)])
    floats = np.array([0.0, -0.0, 1.0, 65504.0, 65520.0, 1e-8, 5.96e-8, 2.98e-8, 6.1e-5, 1023.7, 5000.3, 8190.7,
                       -3.14159, 0.333333, 7.5, 2.0009766], np.float32)
    np.savez_compressed(os.path.join(HERE, "core.npz"), triples=triples, states=np.array(states, np.uint32),
                        seqs=np.array(seqs, np.uint32), floats=floats,
                        halves=np.array([R.lib.sadref_float_to_half(float(f)) for f in floats], np.uint16))

    # candidates: full + warm refresh (test_candidates.cpp:122-168 fixture), both precisions
    st = random_sites(24, 16, 40, 99)
    st.deactivate(3)
    d = sites_dict(st)
    for fp64, opts in ((0, F32), (1, F64)):
        f = sad.CandidateField()
        f.resize(24, 16, 8)
        R.refresh(st, f, sad.RefreshMode.Full, 4, 4, 1234, opts)
        d[f"full_{fp64}"] = f.ids.copy()
        R.refresh(st, f, sad.RefreshMode.WarmStart, 2, 4, 77, opts)
        d[f"warm_{fp64}"] = f.ids.copy()
        d[f"pass_index_{fp64}"] = np.array([f.pass_index])
    np.savez_compressed(os.path.join(HERE, "refresh.npz"), **d)

    # render + backward (test_render.cpp / test_grad.cpp fixtures)
    st = random_model(64, 48, 90, 7)
    tgt = random_target(64, 48, 8)
    f = sad.CandidateField()
    f.resize(64, 48, 8)
    R.refresh(st, f, sad.RefreshMode.Full, 4, 4, 7, F32)
    d = sites_dict(st)
    d.update(ids=f.ids.copy(), target=tgt.data.copy())
    for fp64, opts in ((0, F32), (1, F64)):
        d[f"render_{fp64}"] = R.render_image(st, f, opts).data.copy()
        g = sad.GradBuffer()
        d[f"loss_{fp64}"] = np.array([R.backward_image(st, f, tgt, g, opts, True)])
        d[f"grads_{fp64}"] = g.data.copy()
    d["id_map"] = R.render_id_map(st, f)
    np.savez_compressed(os.path.join(HERE, "render_grad.npz"), **d)

    # stats / prune / densify (test_budget.cpp fixture)
    st = random_model(48, 48, 40, 11)
    tgt = random_target(48, 48, 12)
    f = sad.CandidateField()
    f.resize(48, 48, 8)
    R.refresh(st, f, sad.RefreshMode.Full, 4, 4, 7, F64)
    s = R.accumulate_stats(st, f, tgt)
    d = sites_dict(st)
    d.update(ids=f.ids.copy(), target=tgt.data.copy(), stats=s.data.copy(), valid=np.array([s.valid_pixels]))
    a = st.copy()
    d["pruned"] = np.array([R.prune(a, s, 0.2)])
    adam = sad.AdamState(a.size())
    adam.m[:] = 0.5
    d["densified"] = np.array([R.densify(a, adam, s, tgt, 0.5, sad.TrainConfig())])
    d.update(sites_dict(a, "out_"))
    d["adam_m"] = adam.m.copy()
    np.savez_compressed(os.path.join(HERE, "budget.npz"), **d)

    # init_sites + 3 Adam steps (test_train.cpp fixtures)
    tgt = ramp_image(40, 32)
    cfg = sad.TrainConfig()
    st = sad.SiteStore()
    R.init_sites(st, tgt, 50, cfg)
    d = sites_dict(st, "init_")
    rng = np.random.default_rng(3)
    g = sad.GradBuffer(st.size())
    g.data[:] = rng.normal(size=g.data.shape) * 1e-3
    g.data[5, 0] = np.nan
    st.frozen[7] = 1
    m = sad.AdamState(st.size())
    for _ in range(3):
        R.adam_step(st, g, m, 40, 32, cfg)
    d.update(sites_dict(st, "adam_"))
    d.update(grads=g.data.copy(), m=m.m.copy(), v=m.v.copy(), skipped=np.array([m.skipped]))
    np.savez_compressed(os.path.join(HERE, "train.npz"), **d)

    # a small budgeted fit: full history, final map
    tgt = synth_target(32, 24, 2)
    cfg = sad.TrainConfig(iters=60, target_bpp=4.0, fp64=False, seed=5, densify_start=10, densify_every=10,
                          prune_start=20, prune_every=20)
    r = R.fit(tgt, cfg)
    np.savez_compressed(os.path.join(HERE, "fit.npz"), target=tgt.data.copy(),
                        loss=np.array([h.loss for h in r.history]), psnr=np.array([h.psnr for h in r.history]),
                        active=np.array([h.active_sites for h in r.history]), ids=r.field.ids.copy(),
                        scale=np.array([r.schedule_scale]), **sites_dict(r.sites, "out_"))
    print("golden vectors written to", HERE)


if __name__ == "__main__":
    main()
