"""ctypes mirrors of the POD structs in include/sad_b200.h.

These are layout-only definitions shared by every consumer of the C ABI (the product backend in
`api.py`, and the test-only oracle bindings).  Field order must match the header exactly.
"""
from __future__ import annotations

import ctypes as C

SAD_OK, SAD_EINVAL, SAD_ESTALE, SAD_EEMPTY, SAD_ENUMERIC, SAD_EFORMAT, SAD_ECUDA, SAD_ENOMEM = range(8)
EMPTY_ID = 0xFFFFFFFF

_dp = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)


class SitesView(C.Structure):
    _fields_ = [
        ("size", C.c_size_t),
        ("capacity", C.c_size_t),
        ("x", _dp), ("y", _dp), ("log_tau", _dp), ("radius", _dp),
        ("col_r", _dp), ("col_g", _dp), ("col_b", _dp),
        ("dir_x", _dp), ("dir_y", _dp), ("aniso", _dp),
        ("active", _u8p), ("frozen", _u8p),
        ("generation", C.c_uint64),
    ]


class FieldView(C.Structure):
    _fields_ = [
        ("width", C.c_int), ("height", C.c_int), ("cell", C.c_int),
        ("gw", C.c_int), ("gh", C.c_int), ("k", C.c_int),
        ("ids", C.POINTER(C.c_uint32)),
        ("synced_generation", C.c_uint64),
        ("refresh_count", C.c_uint64),
        ("pass_index", C.c_uint32),
    ]


class PassSpec(C.Structure):
    _fields_ = [("step", C.c_uint32), ("stencil", C.c_int32)]


class AdamView(C.Structure):
    _fields_ = [
        ("sites", C.c_size_t), ("capacity", C.c_size_t),
        ("m", _dp), ("v", _dp),
        ("t", C.c_int64), ("skipped", C.c_uint64),
    ]


class TrainConfigC(C.Structure):
    _fields_ = [
        ("iters", C.c_int32), ("n_sites", C.c_int32), ("target_bpp", C.c_double),
        ("seed", C.c_uint64), ("k", C.c_int32), ("inject", C.c_int32), ("lambda_init", C.c_double),
        ("lr_pos", C.c_double), ("lr_color", C.c_double), ("lr_log_tau", C.c_double),
        ("lr_radius", C.c_double), ("lr_dir", C.c_double), ("lr_aniso", C.c_double),
        ("beta1", C.c_double), ("beta2", C.c_double), ("adam_eps", C.c_double),
        ("refresh_every", C.c_int32), ("refresh_passes", C.c_int32), ("final_passes", C.c_int32),
        ("tau_diffusion_lambda", C.c_double),
        ("densify_every", C.c_int32), ("densify_start", C.c_int32), ("densify_end", C.c_int32),
        ("densify_pct", C.c_double), ("alpha", C.c_double), ("stats_eps", C.c_double),
        ("prune_every", C.c_int32), ("prune_start", C.c_int32), ("prune_end", C.c_int32),
        ("prune_pct", C.c_double), ("prune_during_densify", C.c_int32),
        ("budget_scale_cap", C.c_double), ("max_sites", C.c_uint64),
        ("init_log_tau", C.c_double), ("init_radius", C.c_double), ("init_aniso", C.c_double),
        ("log_tau_min", C.c_double), ("log_tau_max", C.c_double),
        ("radius_min", C.c_double), ("radius_max", C.c_double),
        ("aniso_min", C.c_double), ("aniso_max", C.c_double),
        ("clamp_color", C.c_int32), ("fp64", C.c_int32), ("threads", C.c_int32),
    ]


class HistoryRowC(C.Structure):
    _fields_ = [
        ("iter", C.c_int32), ("loss", C.c_double), ("psnr", C.c_double),
        ("active_sites", C.c_int32), ("ms", C.c_double),
    ]
