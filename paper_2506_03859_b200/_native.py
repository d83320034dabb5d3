"""ctypes binding of libfarqb.so (include/farqb.h).

The product has exactly one compute path: the sm_100a kernels in this .so.  If
the library is missing this module raises -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "lib", "libfarqb.so")


class SketchSpecC(C.Structure):
    _fields_ = [("kind", C.c_int), ("p", C.c_double), ("seed", C.c_uint64), ("zeta", C.c_int)]


class ConfigC(C.Structure):
    _fields_ = [("eps", C.c_double), ("power", C.c_int), ("block", C.c_int), ("sketch", SketchSpecC),
                ("max_iters", C.c_int), ("shift_convention", C.c_int), ("relative", C.c_int)]


class BlockC(C.Structure):
    _fields_ = [("is_dense", C.c_int), ("rows", C.c_int), ("cols", C.c_int),
                ("dense", C.c_void_p), ("col_ptr", C.c_void_p), ("row_idx", C.c_void_p),
                ("values", C.c_void_p), ("nnz", C.c_int64), ("centered", C.c_int),
                ("p", C.c_double), ("std_scale", C.c_double)]


class ResultC(C.Structure):
    _fields_ = [("status", C.c_int), ("m", C.c_int64), ("n", C.c_int64), ("rank", C.c_int),
                ("blocks", C.c_int), ("converged", C.c_int), ("residual_sq", C.c_double),
                ("norm_a_sq", C.c_double), ("q", C.c_void_p), ("ldq", C.c_int64),
                ("bt", C.c_void_p), ("ldbt", C.c_int64), ("on_device", C.c_int),
                ("block_residuals", C.POINTER(C.c_double)), ("block_ids", C.POINTER(C.c_int)),
                ("n_ids", C.c_int), ("resolved_block", C.c_int), ("resolved_max_iters", C.c_int),
                ("resolved_p", C.c_double), ("gpu_launches", C.c_int), ("elapsed_ms", C.c_double),
                ("svd_rank", C.c_int), ("sigma", C.POINTER(C.c_double)), ("v_flagged", C.POINTER(C.c_char)),
                ("u", C.c_void_p), ("ldu", C.c_int64), ("v", C.c_void_p), ("ldv", C.c_int64),
                ("svd_residual_sq", C.c_double), ("internal", C.c_void_p)]


class SketchHostC(C.Structure):
    _fields_ = [("is_dense", C.c_int), ("rows", C.c_int), ("cols", C.c_int),
                ("dense", C.POINTER(C.c_double)), ("col_ptr", C.POINTER(C.c_int)),
                ("row_idx", C.POINTER(C.c_int)), ("values", C.POINTER(C.c_double)),
                ("nnz", C.c_int64), ("centered", C.c_int), ("p", C.c_double),
                ("std_scale", C.c_double)]


SOURCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(BlockC))
HOST_ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int64)

OUT_NONE, OUT_HOST, OUT_DEVICE, OUT_SVD = 0, 1, 2, 4

# every function include/farqb.h declares: (name, restype, argtypes)
_H = C.c_void_p
SIGNATURES = [
    ("fqb_abi_version", C.c_int, []),
    ("fqb_create", C.c_int, [C.c_int, C.POINTER(_H)]),
    ("fqb_destroy", C.c_int, [_H]),
    ("fqb_set_stream", C.c_int, [_H, C.c_void_p]),
    ("fqb_synchronize", C.c_int, [_H]),
    ("fqb_last_error", C.c_char_p, []),
    ("fqb_status_name", C.c_char_p, [C.c_int]),
    ("fqb_launch_count", C.c_int64, [_H]),
    ("fqb_set_pass_timing", C.c_int, [_H, C.c_int]),
    ("fqb_pass_timing", C.c_int, [_H, C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_double)]),
    ("fqb_qb_fixed_precision", C.c_int, [_H, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int,
                                         C.POINTER(ConfigC), SOURCE_FN, C.c_void_p, C.c_uint,
                                         C.POINTER(ResultC)]),
    ("fqb_qb_fixed_rank", C.c_int, [_H, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_int,
                                    C.POINTER(ConfigC), SOURCE_FN, C.c_void_p, C.c_uint,
                                    C.POINTER(ResultC)]),
    ("fqb_qb_fixed_precision_f32", C.c_int, [_H, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int,
                                         C.POINTER(ConfigC), SOURCE_FN, C.c_void_p, C.c_uint,
                                         C.POINTER(ResultC)]),
    ("fqb_qb_fixed_rank_f32", C.c_int, [_H, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_int,
                                    C.POINTER(ConfigC), SOURCE_FN, C.c_void_p, C.c_uint,
                                    C.POINTER(ResultC)]),
    ("fqb_host_free", None, [C.c_void_p]),
    ("fqb_result_free", None, [C.POINTER(ResultC)]),
    ("fqb_comm_unique_id", C.c_int, [C.c_void_p]),
    ("fqb_comm_attach", C.c_int, [_H, C.c_void_p, C.c_int, C.c_int]),
    ("fqb_comm_attach_host", C.c_int, [_H, HOST_ALLREDUCE_FN, C.c_void_p, C.c_int, C.c_int]),
    ("fqb_comm_detach", C.c_int, [_H]),
    ("fqb_collective_count", C.c_int64, [_H]),
    ("fqb_philox_u32", C.c_int, [_H, C.c_uint64, C.c_uint32, C.c_uint32, C.c_int, C.c_void_p]),
    ("fqb_gen_sketch", C.c_int, [_H, C.POINTER(SketchSpecC), C.c_int, C.c_int, C.c_int,
                                 C.POINTER(SketchHostC)]),
    ("fqb_sketch_free", None, [C.POINTER(SketchHostC)]),
    ("fqb_sparse_dense_mul", C.c_int, [_H, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                       C.c_int64]),
    ("fqb_centering_column", C.c_int, [_H, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_double,
                                       C.c_void_p]),
    ("fqb_frob_norm_sq", C.c_int, [_H, C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                                   C.POINTER(C.c_double)]),
    ("fqb_gemm", C.c_int, [_H, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_void_p,
                           C.c_int64, C.c_void_p, C.c_int64, C.c_double, C.c_void_p, C.c_int64]),
    ("fqb_relative_error", C.c_int, [_H, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_void_p,
                                     C.c_int64, C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int,
                                     C.POINTER(C.c_double)]),
    ("fqb_sym_eig", C.c_int, [_H, C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_void_p, C.c_int64,
                              C.POINTER(C.c_int)]),
    ("fqb_gram", C.c_int, [_H, C.c_void_p, C.c_int64, C.c_int, C.c_int64, C.c_void_p, C.c_int64]),
    ("fqb_mul_upper", C.c_int, [_H, C.c_void_p, C.c_int64, C.c_int, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                                C.c_int64]),
    ("fqb_chol_factor", C.c_int, [_H, C.c_void_p, C.c_int, C.c_int64, C.c_double, C.c_double, C.c_void_p,
                                  C.c_int64, C.c_void_p, C.c_int64, C.POINTER(C.c_int)]),
    ("fqb_set_fp32_slices", C.c_int, [_H, C.c_int]),
    ("fqb_fp64_slices", C.c_int, []),
    ("fqb_random_orthonormal", C.c_int, [_H, C.c_int64, C.c_int, C.c_uint64, C.c_uint32, C.c_void_p, C.c_int64]),
    ("fqb_gen_synthetic", C.c_int, [_H, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_void_p, C.c_int64,
                                    C.POINTER(C.c_int)]),
    ("fqb_gen_lowrank", C.c_int, [_H, C.c_int64, C.c_int64, C.c_int, C.c_void_p, C.c_uint64, C.c_double,
                                  C.c_void_p, C.c_int64]),
    ("fqb_host_pool_trim", C.c_size_t, []),
    ("fqb_device_cache_trim", C.c_size_t, []),
    ("fqb_raw_header", C.c_int, [C.c_char_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    ("fqb_load_raw_rows", C.c_int, [_H, C.c_char_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int64, C.c_int,
                                    C.POINTER(C.c_int64)]),
    ("fqb_gen_lowrank_det", C.c_int, [_H, C.c_int64, C.c_int64, C.c_int, C.c_void_p, C.c_uint64, C.c_double,
                                      C.c_int64, C.c_int64, C.c_void_p, C.c_int64]),
    ("fqb_checksum", C.c_int, [_H, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                               C.POINTER(C.c_uint64)]),
    ("fqb_gemm_emulated", C.c_int, [_H, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_void_p,
                                    C.c_int64, C.c_void_p, C.c_int64, C.c_double, C.c_void_p, C.c_int64]),
    ("fqb_slice_operand", C.c_int, [_H, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.POINTER(C.c_void_p)]),
    ("fqb_sliced_gemm", C.c_int, [_H, C.c_void_p, C.c_int, C.c_int64, C.c_double, C.c_void_p, C.c_int64,
                                  C.c_double, C.c_void_p, C.c_int64]),
    ("fqb_sliced_free", C.c_int, [_H, C.c_void_p]),
    ("fqb_sliced_gemm_again", C.c_int, [_H, C.c_void_p, C.c_double, C.c_double, C.c_void_p, C.c_int64]),
    ("fqb_sliced_gemm_mn", C.c_int, [_H, C.c_void_p, C.c_int64, C.c_double, C.c_void_p, C.c_int64, C.c_double,
                                     C.c_void_p, C.c_int64]),
    ("fqb_default_density", C.c_double, [C.c_int, C.c_int64]),
    ("fqb_default_block", C.c_int, [C.c_int64, C.c_int64]),
    ("fqb_default_max_iters", C.c_int, [C.c_int64, C.c_int]),
]

_lib = None


def lib() -> C.CDLL:
    """Load libfarqb.so (built by paper_2506_03859_b200.build / __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build the sm_100a library first "
                "(python -m paper_2506_03859_b200.build). There is no CPU fallback.")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib
