"""Builds an ablation variant of the library: python tools/build_variant.py TAG [-DMACRO=V ...] -> exp/libsad_TAG.so"""
import os, subprocess, sys
sys.path.insert(0, "/root/repo")
import __graft_entry__ as g
tag, defs = sys.argv[1], sys.argv[2:]
d = f"/root/repo/exp/b_{tag}"; os.makedirs(d, exist_ok=True)
objs = []
for s in g.SOURCES:
    o = f"{d}/{s}.o"; objs.append(o)
    subprocess.run([g.NVCC, *g.FLAGS, *defs, "-I", "/root/repo/include", "-c", f"{g.CSRC}/{s}", "-o", o], check=True)
subprocess.run([g.NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", f"/root/repo/exp/libsad_{tag}.so", *objs, "-lcudart"], check=True)
print("ok", tag)
