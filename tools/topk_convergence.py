"""Top-K propagation convergence table (Table "Top-K propagation
convergence (Top-8 exact match)"), with the GPU brute-force checker `exact_topk_batch`
(candidates.cpp:198-248 -> k_exact_topk).

For each domain (1024^2, 2048^2), site count (16k, 65k, 131k) and pass budget (8, 12, 16): collision-free
sites (unique pixel cells plus subpixel offsets, the test fixture of test_candidates.cpp:15-33), the field
seeded by jfa_seed and then `schedule_passes(P)` (candidates.cpp:50-62: Box3 floods at halving steps, then
Axial step-1 passes) with the default injection J = 4; 256 random pixels per trial, 4 trials; the
fraction of pixels whose top-8 set equals the exact top-8 under the (unpacked, fp32) rendering score.

One cell (1024^2, 16k sites, 8 passes, trial 0) is also run on the compiled reference (propagation and
exact_topk on the host) and must give the identical map and the identical exact lists.

    python tools/topk_convergence.py [--trials 4] [--no-ref-check]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2604_21984_b200 as sad  # noqa: E402
from paper_2604_21984_b200.synth import Rng  # noqa: E402

PAPER = {
    (1024, 16384): (0.963, 0.970, 0.970), (1024, 65536): (0.398, 0.867, 0.867), (1024, 131072): (0.072, 0.782, 0.782),
    (2048, 16384): (0.981, 0.987, 0.987), (2048, 65536): (0.393, 0.956, 0.956), (2048, 131072): (0.059, 0.907, 0.907),
}
PASSES = (8, 12, 16)


def collision_free_sites(w, h, n, seed):
    """test_candidates.cpp:15-33 (random_sites), vectorised: a partial Fisher-Yates over the cells with the
    fixture's own seeded stream, then subpixel offsets in [0.25, 0.75)."""
    rng = Rng(seed, 0xC0FFEE, 0)
    cells = np.arange(w * h, dtype=np.int64)
    xs = np.empty(n)
    ys = np.empty(n)
    for i in range(n):
        j = i + rng.next_below(w * h - i)
        cells[i], cells[j] = cells[j], cells[i]
        xs[i] = min((cells[i] % w) + rng.next_unit() * 0.5 + 0.25, w - 1.0)
        ys[i] = min((cells[i] // w) + rng.next_unit() * 0.5 + 0.25, h - 1.0)
    st = sad.SiteStore(n)
    st.x[:] = xs
    st.y[:] = ys
    st.log_tau[:] = 7.5
    st.radius[:] = np.sqrt(w * h / n)
    st.active[:] = 1
    st.bump()
    return st


def probe_pixels(w, h, seed, count=256):
    rng = Rng(seed, 9, 9)
    return np.array([[rng.next_below(w), rng.next_below(h)] for _ in range(count)], np.int32)


def match_fraction(field_ids, w, exact, pix):
    ids = field_ids.reshape(-1, 8)
    hit = 0
    for i, (x, y) in enumerate(pix):
        lst = ids[y * w + x]
        have = set(int(v) for v in lst if v != sad.CandidateField.kEmpty)
        want = set(int(v) for v in exact[i] if v != sad.CandidateField.kEmpty)
        hit += have == want
    return hit / len(pix)


def one(B, W, n, P, trial, schedule):
    st = collision_free_sites(W, W, n, 1000 + trial)
    f = sad.CandidateField()
    f.resize(W, W, 8)
    B.jfa_seed(st, f)
    B.run_passes(st, f, schedule(W, W, P), 4, 77 + trial, sad.RunOpts(fp64=False))
    pix = probe_pixels(W, W, 31 + trial)
    exact = B.exact_topk_batch(st, pix, 8, sad.normalization_scale(W, W), False)
    return st, f, pix, exact


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=4)
    ap.add_argument("--no-ref-check", action="store_true")
    a = ap.parse_args()
    G = sad.gpu_backend(0)
    rows = []
    t0 = time.perf_counter()
    for (W, n), paper in PAPER.items():
        vals = []
        for P in PASSES:
            fr = []
            for trial in range(a.trials):
                st, f, pix, exact = one(G, W, n, P, trial, G.schedule_passes)
                fr.append(match_fraction(f.ids, W, exact, pix))
            vals.append(float(np.mean(fr)))
        rows.append({"domain": W, "sites": n, "top8_exact_match": dict(zip(map(str, PASSES), vals)),
                     "paper": dict(zip(map(str, PASSES), paper))})
        print(f"{W}^2 {n // 1024}k: " + "  ".join(f"{P} passes {v:.3f} (paper {p:.3f})"
                                                  for P, v, p in zip(PASSES, vals, paper)), flush=True)
    out = {"table": rows, "trials": a.trials, "probes_per_trial": 256, "gpu_seconds_total": time.perf_counter() - t0}
    if not a.no_ref_check:
        from oracle.bindings import have_ref, ref_backend
        if have_ref():
            R = ref_backend(threads=os.cpu_count() or 1)
            st, fg, pix, eg = one(G, 1024, 16384, 8, 0, G.schedule_passes)
            _, fr_, _, er = one(R, 1024, 16384, 8, 0, G.schedule_passes)
            same_map = bool(np.array_equal(fg.ids, fr_.ids))
            same_exact = bool(np.array_equal(eg, er))
            out["reference_check"] = {"case": "1024^2, 16k sites, 8 passes, trial 0", "map_identical": same_map,
                                      "exact_lists_identical": same_exact}
            print(f"reference check (1024^2, 16k, 8 passes): map identical {same_map}, exact lists identical "
                  f"{same_exact}", flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
