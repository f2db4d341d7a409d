"""fp64 config-2 divergence probe: fit to iteration T on the GPU and on the reference (all host threads),
compare the states, then replay iteration T+1's warm pass and backward from the reference state on both
libraries and report the per-site gradient differences.   python tools/fp64_div_probe.py [T]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2604_21984_b200 as sad  # noqa: E402
from oracle.bindings import ref_backend  # noqa: E402
from paper_2604_21984_b200.synth import synthetic_image  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 1080
img = sad.ImageBuffer(768, 512, synthetic_image(768, 512, 1))
G = sad.gpu_backend(0)
R = ref_backend(threads=os.cpu_count() or 1)
states = {}
for name, B, env in (("gpu", G, "SAD_STOP_AT"), ("ref", R, "SAD_REF_STOP_AT")):
    os.environ[env] = str(T)
    cfg = sad.TrainConfig(iters=4000, target_bpp=2.0, fp64=True, seed=1)
    cfg.threads = os.cpu_count() or 1
    states[name] = B.fit(img, cfg)
    del os.environ[env]
a, b = states["gpu"], states["ref"]
print("pass_index", a.field.pass_index, b.field.pass_index, "sites", a.sites.size(), b.sites.size())
print("ids identical", np.array_equal(a.field.ids, b.field.ids), "x identical", np.array_equal(a.sites.x, b.sites.x))
for p in ("x", "y", "log_tau", "radius", "col_r", "dir_x", "aniso", "active"):
    d = np.flatnonzero(getattr(a.sites, p) != getattr(b.sites, p))
    print(p, "differs at", d[:12], [(getattr(a.sites, p)[i], getattr(b.sites, p)[i]) for i in d[:3]])
print("history identical", [sad.history_line(r) for r in a.history] == [sad.history_line(r) for r in b.history])
st, f = b.sites, b.field
f.synced_generation = st.generation
opts = sad.RunOpts(fp64=True)
fg, fr = f.copy(), f.copy()
G.refresh(st, fg, sad.RefreshMode.WarmStart, 1, 4, 1, opts)
R.refresh(st, fr, sad.RefreshMode.WarmStart, 1, 4, 1, opts)
print("warm pass maps identical", np.array_equal(fg.ids, fr.ids))
gg, gr = sad.GradBuffer(), sad.GradBuffer()
lg = G.backward_image(st, fr, img, gg, opts, False)
lr = R.backward_image(st, fr, img, gr, opts, False)
print("loss", repr(lg), repr(lr), lg == lr)
d = np.flatnonzero((gg.data.view(np.uint64) != gr.data.view(np.uint64)).any(1))
print("sites with differing gradients:", len(d), d[:20])
for s in d[:8]:
    k = np.flatnonzero(gg.data[s].view(np.uint64) != gr.data[s].view(np.uint64))
    print(s, [(int(c), gg.data[s, c], gr.data[s, c]) for c in k])
# the same backward in fp32 for comparison
gg, gr = sad.GradBuffer(), sad.GradBuffer()
G.backward_image(st, fr, img, gg, sad.RunOpts(fp64=False), False)
R.backward_image(st, fr, img, gr, sad.RunOpts(fp64=False), False)
print("fp32 backward identical:", np.array_equal(gg.data, gr.data))
