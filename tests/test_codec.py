"""The `.sad` container (codec.hpp / codec.cpp): encode/decode byte- and value-identical to the
reference, malformed-input errors, and the device decode pipeline (read -> refresh(Full,16) ->
render) against the reference's."""
import numpy as np
import pytest

import paper_2604_21984_b200 as sad
from oracle.bindings import c_backend, have_ref, ref_backend
from tests.fixtures import random_model

PARAMS = ("x", "y", "log_tau", "radius", "col_r", "col_g", "col_b", "dir_x", "dir_y", "aniso", "active")


def _model():
    st = random_model(64, 48, 70, 21)
    st.deactivate(5)
    return st


def _lib():
    """The product library's codec runs on the host; it loads without a GPU."""
    from paper_2604_21984_b200 import api
    return api.Backend(api.load_library(), "sad_", ctx=None)


@pytest.mark.skipif(not have_ref(), reason="reference library not built")
def test_c_oracle_codec_matches_reference():
    R, O = ref_backend(), c_backend()
    st = _model()
    a, b = R.encode_sites(st, 64, 48), O.encode_sites(st, 64, 48)
    assert a == b and len(a) == 58 + 16 * 69
    wa, ha, sa = R.decode_sites(a)
    wb, hb, sb = O.decode_sites(a)
    assert (wa, ha) == (wb, hb) == (64, 48)
    for p in PARAMS:
        assert np.array_equal(getattr(sa, p), getattr(sb, p)), p


def test_product_codec_matches_oracle():
    O = c_backend()
    try:
        L = _lib()
    except Exception as e:  # pragma: no cover
        pytest.skip(f"library not loadable: {e}")
    st = _model()
    data = O.encode_sites(st, 64, 48)
    assert L.encode_sites(st, 64, 48) == data
    w, h, s2 = L.decode_sites(data)
    _, _, s3 = O.decode_sites(data)
    for p in PARAMS:
        assert np.array_equal(getattr(s2, p), getattr(s3, p)), p
    with pytest.raises(sad.api.FormatError):
        L.decode_sites(data[:-3])
    with pytest.raises(sad.api.FormatError):
        L.decode_sites(b"SADX" + data[4:])


@pytest.mark.gpu
def test_decode_render_pipeline():
    G = sad.gpu_backend(0)
    R = ref_backend() if have_ref() else c_backend()
    st = _model()
    data = R.encode_sites(st, 64, 48)
    img_g, sg = G.decode_render(data, passes=16, seed=3)
    img_r, sr = R.decode_render(data, passes=16, seed=3)
    for p in PARAMS:
        assert np.array_equal(getattr(sg, p), getattr(sr, p)), p
    assert np.array_equal(img_g.data, img_r.data)
