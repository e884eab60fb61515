"""ctypes binding of libstencil_tiler.so (include/stencil_tiler.h).

The library is built in-tree by ``make`` in this directory (or
``__graft_entry__.build()``).  There is no fallback: if the shared object is
missing, importing the executor raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libstencil_tiler.so")
if os.environ.get("ST_EXP_LIB", "0") not in ("", "0"):  # profiling ablation builds (make EXP=n); never the default
    LIB_PATH = os.path.join(_HERE, f"libstencil_tiler_exp{int(os.environ['ST_EXP_LIB'])}.so")

ST_MAX_DIMS = 3


class st_term(C.Structure):
    _fields_ = [("coeff", C.c_float), ("dt", C.c_int), ("offsets", C.c_int * ST_MAX_DIMS)]


class st_plan(C.Structure):
    _fields_ = [
        ("schedule", C.c_int),
        ("skew", C.c_int),
        ("time_tile", C.c_int64),
        ("space_tiles", C.c_int64 * ST_MAX_DIMS),
        ("fused_levels", C.c_int64),
        ("band_rows", C.c_int64),
        ("band_skew", C.c_int),
    ]


class st_report(C.Structure):
    _fields_ = [
        ("points_updated", C.c_int64),
        ("flops", C.c_int64),
        ("wall_seconds", C.c_double),
        ("device_seconds", C.c_double),
        ("time_tile_used", C.c_int64),
        ("kernel_launches", C.c_int64),
        ("tile", C.c_int64 * 3),
        ("mode_used", C.c_int),
        ("kernel_kind", C.c_int),
    ]


class st_traffic(C.Structure):
    _fields_ = [
        ("lines_loaded", C.c_int64),
        ("lines_written_back", C.c_int64),
        ("line_elems", C.c_int64),
        ("bytes", C.c_int64),
        ("flops", C.c_int64),
        ("measured_ai", C.c_double),
    ]


# (name, restype, argtypes) for every symbol declared in include/stencil_tiler.h
P = C.c_void_p
I64P = C.POINTER(C.c_int64)
FP = C.POINTER(C.c_float)
SIGNATURES = [
    ("st_last_error", C.c_char_p, []),
    ("st_version", C.c_char_p, []),
    ("st_stencil_create", C.c_int, [C.c_char_p, C.c_int, C.POINTER(st_term), C.c_int, C.c_int, C.POINTER(P)]),
    ("st_stencil_parse", C.c_int, [C.c_char_p, C.POINTER(P), C.POINTER(C.c_int), I64P, I64P, C.POINTER(C.c_int)]),
    ("st_stencil_destroy", None, [P]),
    ("st_stencil_ndims", C.c_int, [P]),
    ("st_stencil_model", C.c_int, [P]),
    ("st_stencil_nterms", C.c_int, [P]),
    ("st_stencil_term", C.c_int, [P, C.c_int, C.POINTER(st_term)]),
    ("st_stencil_time_depth", C.c_int, [P]),
    ("st_stencil_radius", C.c_int, [P, C.c_int]),
    ("st_min_skew_factor", C.c_int, [P]),
    ("st_time_buffer_slots", C.c_int64, [P, C.c_int64]),
    ("st_flops_per_point", C.c_int64, [P]),
    ("st_check_legality", C.c_int, [P, C.POINTER(st_plan), C.POINTER(C.c_int)]),
    ("st_required_slots", C.c_int64, [P, C.POINTER(st_plan)]),
    ("st_layout_plane", C.c_int64, [P, I64P]),
    ("st_init_reference", C.c_int, [P, I64P, FP, C.c_int64, C.c_uint64]),
    ("st_init_unit", C.c_int, [P, I64P, FP, C.c_int64, C.c_uint64]),
    ("st_init_gaussian", C.c_int, [P, I64P, FP, C.c_int64, C.c_double, I64P]),
    ("st_init_gaussian_slab", C.c_int, [P, I64P, FP, C.c_int64, C.c_double, I64P, C.c_int64]),
    ("st_field_layered", C.c_int, [C.c_int, I64P, FP, C.c_double, C.c_double, C.c_int64, C.c_double, C.c_double, C.c_int64]),
    ("st_field_random_smoothed", C.c_int, [C.c_int, I64P, FP, C.c_uint64, C.c_double, C.c_double, C.c_double, C.c_double]),
    ("st_verify_bitwise", C.c_int, [P, I64P, FP, C.c_int64, FP, C.c_int64, C.c_int64, C.c_int64, C.POINTER(C.c_int)]),
    ("st_verify_bitwise_layout", C.c_int, [C.c_int, I64P, I64P, FP, C.c_int64, FP, C.c_int64, C.c_int64, C.c_int64,
                                           C.POINTER(C.c_int)]),
    ("st_simulate", C.c_int, [P, I64P, C.c_int64, C.POINTER(st_plan), C.c_int64, C.c_int64, C.c_int64,
                              C.POINTER(st_traffic)]),
    ("st_context_create", C.c_int, [C.c_int, C.POINTER(P)]),
    ("st_context_destroy", None, [P]),
    ("st_context_stream", P, [P]),
    ("st_context_device", C.c_int, [P]),
    ("st_context_sm_count", C.c_int, [P]),
    ("st_context_flush_l2", C.c_int, [P]),
    ("st_grid_create", C.c_int, [P, P, I64P, C.c_int64, C.POINTER(P)]),
    ("st_grid_destroy", None, [P]),
    ("st_grid_upload", C.c_int, [P, FP, C.c_int64, C.c_int64, C.c_uint]),
    ("st_grid_set_field", C.c_int, [P, FP, C.c_int64]),
    ("st_grid_download", C.c_int, [P, FP, C.c_int64, I64P]),
    ("st_grid_last_level", C.c_int, [P, I64P]),
    ("st_grid_device_bytes", C.c_int64, [P]),
    ("st_apply", C.c_int, [P, C.c_int64, C.c_int64, C.POINTER(st_plan), C.c_int, C.POINTER(st_report)]),
    ("st_execute_host", C.c_int, [P, FP, C.c_int64, C.c_int64, C.c_int64, C.POINTER(st_plan), C.c_int, C.c_uint,
                                  C.POINTER(st_report)]),
    ("st_dist_partition", C.c_int, [C.c_int64, C.c_int, C.c_int, C.c_int64, I64P, I64P, I64P, I64P]),
    ("st_nccl_unique_id", C.c_int, [C.c_char_p]),
    ("st_dist_create", C.c_int, [P, C.c_int, C.c_int, C.c_char_p, C.c_int64, C.c_int64, C.POINTER(P)]),
    ("st_dist_link_loopback", C.c_int, [C.POINTER(P), C.c_int]),
    ("st_dist_apply", C.c_int, [P, C.c_int64, C.c_int64, C.POINTER(st_plan), C.c_int, C.POINTER(st_report)]),
    ("st_dist_destroy", None, [P]),
]

_lib = None


def load() -> C.CDLL:
    """Load (once) and type the native library; raise if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make -C paper_1806_08299_b200` "
            "or __graft_entry__.build() (there is no CPU fallback)"
        )
    lib = C.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def i64array(vals):
    arr = (C.c_int64 * ST_MAX_DIMS)()
    for i, v in enumerate(vals):
        arr[i] = int(v)
    for i in range(len(vals), ST_MAX_DIMS):
        arr[i] = 1
    return arr
