"""fp64 config-2: stats at the t = T event from the reference state after iteration T-1, on the GPU and on
the reference with 1 and all threads.   python tools/fp64_stats_probe.py [T]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2604_21984_b200 as sad  # noqa: E402
from oracle.bindings import ref_backend  # noqa: E402
from paper_2604_21984_b200.synth import synthetic_image  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 1040
img = sad.ImageBuffer(768, 512, synthetic_image(768, 512, 1))
G = sad.gpu_backend(0)
nt = os.cpu_count() or 1
R = ref_backend(threads=nt)
R1 = ref_backend(threads=1)
os.environ["SAD_REF_STOP_AT"] = str(T - 1)
cfg = sad.TrainConfig(iters=4000, target_bpp=2.0, fp64=True, seed=1)
cfg.threads = nt
b = R.fit(img, cfg)
del os.environ["SAD_REF_STOP_AT"]
st, f = b.sites, b.field
f.synced_generation = st.generation
opts = sad.RunOpts(fp64=True)
R.refresh(st, f, sad.RefreshMode.WarmStart, 1, 4, 1, opts)
s_gpu = G.accumulate_stats(st, f, img)
s_r1 = R1.accumulate_stats(st, f, img)
s_rn = R.accumulate_stats(st, f, img)
for name, s in (("ref 1 thread", s_r1), (f"ref {nt} threads", s_rn)):
    d = np.flatnonzero((s_gpu.data.view(np.uint64) != s.data.view(np.uint64)).any(1))
    print(f"gpu vs {name}: {len(d)} sites differ {d[:10]}")
d = np.flatnonzero((s_r1.data.view(np.uint64) != s_rn.data.view(np.uint64)).any(1))
print(f"ref 1 vs {nt} threads: {len(d)} sites differ {d[:10]}")
dd = np.flatnonzero((s_gpu.data.view(np.uint64) != s_r1.data.view(np.uint64)).any(1))
for i in dd[:4]:
    c = np.flatnonzero(s_gpu.data[i].view(np.uint64) != s_r1.data[i].view(np.uint64))
    print(i, [(int(k), s_gpu.data[i, k], s_r1.data[i, k], s_rn.data[i, k]) for k in c])
for name, B in (("gpu", G), ("ref1", R1), ("refN", R)):
    gb = sad.GradBuffer()
    B.backward_image(st, f, img, gb, opts, False)
    globals()["g_" + name] = gb.data
for name in ("ref1", "refN"):
    d = np.flatnonzero((g_gpu.view(np.uint64) != globals()["g_" + name].view(np.uint64)).any(1))
    print(f"backward gpu vs {name}: {len(d)} sites differ {d[:10]}")
d = np.flatnonzero((g_ref1.view(np.uint64) != g_refN.view(np.uint64)).any(1))
print(f"backward ref1 vs refN: {len(d)} sites differ {d[:10]}")
for i in np.flatnonzero((g_gpu.view(np.uint64) != g_ref1.view(np.uint64)).any(1))[:4]:
    c = np.flatnonzero(g_gpu[i].view(np.uint64) != g_ref1[i].view(np.uint64))
    print(i, [(int(k), g_gpu[i, k], g_ref1[i, k], g_refN[i, k]) for k in c])
np.savez_compressed("gpurun_out/fp64_stats_state.npz", **{p: getattr(st, p) for p in
                    ("x", "y", "log_tau", "radius", "col_r", "col_g", "col_b", "dir_x", "dir_y", "aniso", "active",
                     "frozen")}, ids=f.ids, gen=st.generation)
