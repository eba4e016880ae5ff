"""ctypes binding of libsbx.so (the C-ABI declared in include/sbx.h).

Loading fails loudly when the CUDA library has not been built: there is no
CPU fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "_lib" / "libsbx.so"
if os.environ.get("SBX_LIB_DIR"):  # diagnostics: an alternative in-tree build (e.g. _libexp)
    LIB_PATH = _PKG / os.environ["SBX_LIB_DIR"] / "libsbx.so"

I64 = C.c_int64
I64P = C.POINTER(C.c_int64)
F64P = C.POINTER(C.c_double)
VP = C.c_void_p

SBX_OK = 0
SBX_INVALID_ARGUMENT = 1
SBX_NONCONVERGENCE = 2
SBX_GEOMETRY_ERROR = 3
SBX_SINGULAR_MATRIX = 4
SBX_PROXY_VIOLATION = 5
SBX_CUDA_ERROR = 6
SBX_RUNTIME_ERROR = 7

SBX_TRANSPOSE = 1
SBX_DEVICE_PTRS = 2
SBX_ROW_MAJOR = 4


class sbx_curve(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("center_x", C.c_double),
        ("center_y", C.c_double),
        ("scale", C.c_double),
        ("flip_normal", C.c_int32),
        ("n_prongs", C.c_int32),
        ("amplitude", C.c_double),
        ("aspect", C.c_double),
        ("n_cos", C.c_int32),
        ("n_sin", C.c_int32),
        ("cos_coef", C.c_double * 64),
        ("sin_coef", C.c_double * 64),
    ]


class sbx_hbs_options(C.Structure):
    _fields_ = [
        ("eps", C.c_double),
        ("leaf_nodes", C.c_int64),
        ("n_proxy", C.c_int32),
        ("bas_factor", C.c_double),
        ("div_factor", C.c_double),
    ]


_lib = None

# (name, restype, argtypes)
_SIGS = [
    ("sbx_last_error", C.c_char_p, []),
    ("sbx_init", C.c_int, [C.c_int]),
    ("sbx_sync", C.c_int, []),
    ("sbx_stream", C.c_void_p, []),
    ("sbx_kernel_launches", C.c_int64, [C.c_int]),
    ("sbx_kernel_timing", C.c_int, [C.c_int]),
    ("sbx_kernel_time", C.c_int, [C.c_char_p, C.c_int, C.POINTER(C.c_double), I64P]),
    ("sbx_kernel_flops", C.c_int, [C.c_char_p, C.c_int, C.POINTER(C.c_double)]),
    ("sbx_row_id", C.c_int, [F64P, I64, I64, C.c_double, I64, C.c_int, I64P, I64P, F64P]),
    ("sbx_dense_inverse", C.c_int, [F64P, I64, F64P, C.POINTER(C.c_double)]),
    ("sbx_matmul", C.c_int, [F64P, I64, I64, F64P, I64, F64P]),
    ("sbx_geom_create", C.c_int, [C.POINTER(sbx_curve), C.c_int, C.c_int, C.POINTER(VP)]),
    ("sbx_geom_add_holes", C.c_int,
     [VP, C.c_int, C.POINTER(sbx_curve), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
      C.POINTER(VP), C.POINTER(VP)]),
    ("sbx_geom_destroy", C.c_int, [VP]),
    ("sbx_geom_info", C.c_int, [VP, I64P, I64P, I64P]),
    ("sbx_geom_nodes", C.c_int, [VP, F64P, I64P]),
    ("sbx_panels_near_point", C.c_int, [VP, C.c_double, C.c_double, C.c_double, I64P, I64, I64P]),
    ("sbx_refine", C.c_int, [VP, I64P, I64, C.c_int, C.POINTER(VP), C.POINTER(VP)]),
    ("sbx_coarsen", C.c_int, [VP, VP, C.POINTER(VP)]),
    ("sbx_plan_destroy", C.c_int, [VP]),
    ("sbx_plan_sizes", C.c_int, [VP, I64P, I64P, I64P]),
    ("sbx_plan_maps", C.c_int, [VP, I64P, I64P, I64P, I64P]),
    ("sbx_submatrix", C.c_int, [VP, C.c_int, C.c_double, I64P, I64, I64P, I64, F64P]),
    ("sbx_boundary_data", C.c_int, [VP, I64, F64P, C.c_double, F64P]),
    ("sbx_evaluate_solution", C.c_int,
     [VP, C.c_int, C.c_double, F64P, I64, I64, F64P, I64, C.c_int, F64P, F64P, C.POINTER(C.c_uint8)]),
    ("sbx_hbs_compress", C.c_int, [VP, C.c_int, C.c_double, C.POINTER(sbx_hbs_options), C.POINTER(VP)]),
    ("sbx_hbs_compress_subset", C.c_int,
     [VP, C.c_int, C.c_double, I64P, I64, C.POINTER(sbx_hbs_options), C.POINTER(VP)]),
    ("sbx_hbs_invert", C.c_int, [VP]),
    ("sbx_hbs_destroy", C.c_int, [VP]),
    ("sbx_hbs_solve", C.c_int, [VP, VP, I64, I64, VP, I64, C.c_int, VP]),
    ("sbx_hbs_apply", C.c_int, [VP, VP, I64, I64, VP, I64, C.c_int, VP]),
    ("sbx_hbs_shard_info", C.c_int, [VP, C.c_int, C.c_int, I64P, I64P, I64P]),
    ("sbx_hbs_solve_shard_up", C.c_int, [VP, C.c_int, C.c_int, VP, I64, I64, VP, C.c_int, VP]),
    ("sbx_hbs_solve_shard_down", C.c_int, [VP, C.c_int, C.c_int, VP, I64, VP, I64, C.c_int, VP]),
    ("sbx_hbs_save_hbs1", C.c_int, [VP, C.c_char_p]),
    ("sbx_hbs_load_hbs1", C.c_int, [C.c_char_p, C.POINTER(VP)]),
    ("sbx_hbs_info", C.c_int, [VP, I64P]),
    ("sbx_hbs_node_ranks", C.c_int, [VP, I64P, I64]),
    ("sbx_update_compress", C.c_int,
     [VP, VP, VP, C.c_int, C.c_double, C.c_double, C.c_uint64, C.POINTER(VP)]),
    ("sbx_update_destroy", C.c_int, [VP]),
    ("sbx_update_info", C.c_int, [VP, I64P]),
    ("sbx_update_factor", C.c_int, [VP, C.c_int, F64P]),
    ("sbx_update_from_factors", C.c_int, [VP, F64P, F64P, I64, I64, C.POINTER(VP)]),
    ("sbx_dump_matrix", C.c_int, [C.c_char_p, F64P, I64, I64, I64]),
    ("sbx_hbs_compress_custom", C.c_int, [VP, C.c_int, C.c_double, VP, VP, C.c_int,
                                          C.POINTER(sbx_hbs_options), C.POINTER(VP)]),
    ("sbx_update_compress_mode", C.c_int, [VP, VP, VP, C.c_int, C.c_double, C.c_double, C.c_uint64, C.c_int,
                                           C.POINTER(VP)]),
    ("sbx_els_conditioning_report", C.c_int, [VP, C.c_int, C.c_int, F64P]),
    ("sbx_comm_unique_id", C.c_int, [C.POINTER(C.c_uint8)]),
    ("sbx_hbs_compress_sharded", C.c_int, [VP, C.c_int, C.c_double, C.POINTER(sbx_hbs_options), VP,
                                           C.POINTER(VP)]),
    ("sbx_comm_create", C.c_int, [C.POINTER(C.c_uint8), C.c_int, C.c_int, C.POINTER(VP)]),
    ("sbx_comm_create_loopback", C.c_int, [C.c_int, C.POINTER(VP)]),
    ("sbx_comm_destroy", C.c_int, [VP]),
    ("sbx_comm_info", C.c_int, [VP, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("sbx_hbs_solve_sharded", C.c_int, [VP, VP, VP, I64, I64, VP, I64, C.c_int, VP]),
    ("sbx_els_shard_build", C.c_int, [VP, VP, VP, VP, VP, VP, C.c_int, C.c_double, VP, C.POINTER(VP)]),
    ("sbx_els_shard_info", C.c_int, [VP, I64P]),
    ("sbx_els_shard_rows", C.c_int, [VP, I64P]),
    ("sbx_els_shard_solve", C.c_int, [VP, VP, I64, VP, I64, I64, VP, I64, VP, I64, C.c_int, VP]),
    ("sbx_els_shard_destroy", C.c_int, [VP]),
    ("sbx_update_cache_create", C.c_int, [C.POINTER(VP)]),
    ("sbx_update_cache_destroy", C.c_int, [VP]),
    ("sbx_update_cache_compress", C.c_int, [VP, VP, VP, VP, I64P, I64, C.c_int, C.c_int, C.c_double,
                                            C.c_double, C.c_uint64, C.POINTER(VP), C.POINTER(C.c_int)]),
    ("sbx_update_cache_stats", C.c_int, [VP, I64P, I64P, I64P]),
    ("sbx_load_matrix_dims", C.c_int, [C.c_char_p, I64P, I64P]),
    ("sbx_load_matrix", C.c_int, [C.c_char_p, F64P, I64]),
    ("sbx_update_dump", C.c_int, [VP, C.c_char_p, C.c_char_p]),
    ("sbx_update_load", C.c_int, [VP, C.c_char_p, C.c_char_p, C.POINTER(VP)]),
    ("sbx_els_build", C.c_int, [VP, VP, VP, VP, VP, C.c_int, C.c_double, C.POINTER(VP)]),
    ("sbx_els_destroy", C.c_int, [VP]),
    ("sbx_els_info", C.c_int, [VP, I64P]),
    ("sbx_els_solve", C.c_int, [VP, VP, I64, I64, VP, I64, C.c_int, VP]),
    ("sbx_els_solve_raw", C.c_int, [VP, VP, I64, I64, VP, I64, C.c_int, VP]),
    ("sbx_els_density_on_refined", C.c_int, [VP, F64P, F64P]),
    ("sbx_els_apply_forward", C.c_int, [VP, F64P, I64, I64, F64P, I64]),
    ("sbx_els_apply_forward_t", C.c_int, [VP, F64P, I64, I64, F64P, I64]),
    ("sbx_els_conditioning", C.c_int, [VP, C.c_int, F64P]),
    ("sbx_els_gmres", C.c_int, [VP, F64P, F64P, C.c_int, C.c_double, I64, I64, I64P, F64P, I64]),
    ("sbx_els_xw", C.c_int, [VP, F64P, F64P]),
    ("sbx_app_build", C.c_int, [VP, VP, C.c_int, C.c_double, C.c_double, C.POINTER(VP)]),
    ("sbx_app_destroy", C.c_int, [VP]),
    ("sbx_app_info", C.c_int, [VP, I64P]),
    ("sbx_app_solve", C.c_int, [VP, VP, I64, I64, VP, I64, C.c_int, VP]),
]

EXPORTS = [s[0] for s in _SIGS]


def lib():
    """Load libsbx.so (raises if the CUDA extension was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA library first "
                "(python -c 'import __graft_entry__ as g; g.build()'); "
                "this package has no CPU fallback")
        L = C.CDLL(str(LIB_PATH))
        for name, res, args in _SIGS:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class SbxError(RuntimeError):
    code = SBX_RUNTIME_ERROR


class GeometryError(SbxError):
    code = SBX_GEOMETRY_ERROR


class SingularMatrixError(SbxError):
    code = SBX_SINGULAR_MATRIX


class ProxyViolationError(SbxError):
    code = SBX_PROXY_VIOLATION


class CudaError(SbxError):
    code = SBX_CUDA_ERROR


class ConvergenceError(SbxError):
    code = SBX_NONCONVERGENCE


def check(code: int):
    if code == SBX_OK:
        return
    msg = lib().sbx_last_error().decode(errors="replace")
    if code == SBX_INVALID_ARGUMENT:
        raise ValueError(msg)
    cls = {SBX_GEOMETRY_ERROR: GeometryError, SBX_SINGULAR_MATRIX: SingularMatrixError,
           SBX_PROXY_VIOLATION: ProxyViolationError, SBX_CUDA_ERROR: CudaError,
           SBX_NONCONVERGENCE: ConvergenceError}.get(code, SbxError)
    raise cls(msg)
