"""The C-ABI boundary (CPU-only): libsad_b200.so loads without a GPU and exports every function
declared in include/sad_b200.h; the ctypes struct mirrors match the header's layout; host-only
entry points (schedule helpers, codec) behave like the reference."""
import ctypes as C
import os
import re

import pytest

from paper_2604_21984_b200 import _abi, api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sad_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sad_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = api.load_library()
    missing = [f for f in declared_functions() if not hasattr(lib, f)]
    assert not missing, missing
    assert len(declared_functions()) >= 45
    assert lib.sad_abi_version() == 1


def test_struct_layouts():
    # sizes fixed by the header's field order (x86-64 / aarch64 LP64 alignment)
    assert C.sizeof(_abi.SitesView) == 8 * 2 + 8 * 12 + 8
    assert C.sizeof(_abi.FieldView) == 6 * 4 + 8 + 8 + 8 + 4 + 4
    assert C.sizeof(_abi.TrainConfigC) == 312
    lib = api.load_library()
    c = _abi.TrainConfigC()
    lib.sad_default_config(C.byref(c))
    import paper_2604_21984_b200 as sad
    d = sad.TrainConfig().to_c()
    assert bytes(c)[:C.sizeof(c)] == bytes(d)[:C.sizeof(d)]


def test_host_entry_points_without_gpu():
    import paper_2604_21984_b200 as sad
    B = api.Backend(api.load_library(), "sad_", ctx=None)
    assert B.jump_step(7, 2048) == 8
    assert [p.step for p in B.full_refresh_passes(768, 512, 4)] == [512, 256, 128, 64, 32, 16, 8, 4, 2, 1, 1, 1, 1, 1]
    assert B.bpp_target_count(2.0, 768, 512) == 6144
    assert abs(B.plan_schedule(9831, 6144, sad.TrainConfig()) - 0.49865722656250006) < 1e-15
    with pytest.raises(sad.InvalidArgument):
        B.jump_step(0, 1000)


@pytest.mark.gpu
def test_library_refuses_without_matching_device():
    import paper_2604_21984_b200 as sad
    G = sad.gpu_backend(0)
    assert G.ctx
