"""ctypes binding of libnpsd_b200.so (include/npsd_b200.h). No fallback: if the
library is missing the import of the product path fails loudly."""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

# NPSD_B200_LIB: another build of the same library (A/B measurements of compile-time variants)
LIB_PATH = Path(os.environ.get("NPSD_B200_LIB") or Path(__file__).resolve().parent / "libnpsd_b200.so")

NPSD_OK, NPSD_INVALID_ARGUMENT, NPSD_BREAKDOWN, NPSD_EMPTY_SYSTEM, NPSD_CUDA_ERROR, NPSD_IO_ERROR = range(6)

EXPORTED_SYMBOLS = (
    "npsd_b200_create", "npsd_b200_destroy", "npsd_b200_last_error", "npsd_b200_set_params",
    "npsd_b200_set_mask", "npsd_b200_set_mask_device", "npsd_b200_n_fluid", "npsd_b200_fluid_indices",
    "npsd_b200_precond_apply", "npsd_b200_psdo_solve", "npsd_b200_psdo_solve_n", "npsd_b200_psdo_solve_device", "npsd_b200_spmv",
    "npsd_b200_net_apply", "npsd_b200_level_image", "npsd_b200_linear_coeffs", "npsd_b200_mixed_counts",
    "npsd_b200_param_count", "npsd_b200_init_params", "npsd_b200_identity_params", "npsd_b200_rhs_normal",
    "npsd_b200_device_alloc", "npsd_b200_device_free", "npsd_b200_host_alloc", "npsd_b200_host_free",
    "npsd_b200_memcpy", "npsd_b200_synchronize", "npsd_b200_last_solve_ms", "npsd_b200_last_solve_launches",
    "npsd_b200_launch_count", "npsd_b200_event_record", "npsd_b200_event_elapsed_ms",
    "npsd_b200_profile_iterations", "npsd_b200_save_npm", "npsd_b200_load_npm", "npsd_b200_npm_last_error",
    "npsd_b200_nccl_unique_id", "npsd_b200_comm_create_nccl", "npsd_b200_comm_create_local",
    "npsd_b200_comm_destroy", "npsd_b200_comm_last_error", "npsd_b200_create_slab", "npsd_b200_slab_graph",
    "npsd_b200_mac_divergence_rhs", "npsd_b200_mac_divergence_rhs_device", "npsd_b200_pcg_solve",
    "npsd_b200_pcg_solve_device", "npsd_b200_ic0_apply", "npsd_b200_is_pure_neumann", "npsd_b200_check_operator",
    "npsd_b200_set_exact",
)


class SolveCfg(C.Structure):
    _fields_ = [("tol_reduction", C.c_double), ("tol_abs", C.c_double), ("max_iters", C.c_int64),
                ("n_ortho", C.c_int32), ("nullspace_projection", C.c_int32),
                ("normalize_before_precond", C.c_int32), ("precond", C.c_int32)]


class Report(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("converged", C.c_int32), ("breakdown", C.c_int32),
                ("residual_history", C.POINTER(C.c_double)), ("cumulative_seconds", C.POINTER(C.c_double)),
                ("history_len", C.c_int64), ("setup_seconds", C.c_double), ("iterate_seconds", C.c_double),
                ("precond_seconds", C.c_double)]


_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_vp = C.c_void_p

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} is not built (run __graft_entry__.build()); the B200 path has no CPU fallback")
    L = C.CDLL(str(LIB_PATH))
    L.npsd_b200_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _f32p, C.c_size_t, C.c_void_p,
                                   C.c_int, C.POINTER(_vp)]
    L.npsd_b200_destroy.argtypes = [_vp]
    L.npsd_b200_last_error.restype = C.c_char_p
    L.npsd_b200_comm_last_error.restype = C.c_char_p
    L.npsd_b200_comm_last_error.argtypes = []
    L.npsd_b200_nccl_unique_id.argtypes = [C.c_void_p]
    L.npsd_b200_comm_create_nccl.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(_vp)]
    L.npsd_b200_comm_create_local.argtypes = [C.c_int, C.POINTER(_vp)]
    L.npsd_b200_comm_destroy.argtypes = [_vp]
    L.npsd_b200_slab_graph.argtypes = [_vp]
    L.npsd_b200_pcg_solve.argtypes = [_vp, _f64p, _vp, C.c_void_p, C.c_int, _f64p, C.c_void_p]
    L.npsd_b200_pcg_solve_device.argtypes = [_vp, _vp, _vp, C.c_void_p, C.c_int, _vp, C.c_void_p]
    L.npsd_b200_ic0_apply.argtypes = [_vp, _f64p, _f64p, C.c_int64, C.POINTER(C.c_int)]
    L.npsd_b200_mac_divergence_rhs.argtypes = [_vp, _vp, _vp, _vp, C.c_double, C.c_double, C.c_double, _vp, _vp,
                                               _vp, _vp]
    L.npsd_b200_mac_divergence_rhs_device.argtypes = [_vp, _vp, _vp, _vp, C.c_double, C.c_double, C.c_double, _vp,
                                                      _vp, _vp, _vp]
    L.npsd_b200_create_slab.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _f32p, C.c_size_t,
                                        C.c_int, _vp, C.c_int, C.POINTER(_vp)]
    L.npsd_b200_npm_last_error.restype = C.c_char_p
    L.npsd_b200_npm_last_error.argtypes = []
    L.npsd_b200_save_npm.argtypes = [C.c_char_p, C.c_int, C.c_int, _f32p, C.c_size_t]
    L.npsd_b200_load_npm.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_void_p, C.c_size_t,
                                     C.POINTER(C.c_size_t)]
    L.npsd_b200_last_error.argtypes = [_vp]
    L.npsd_b200_set_params.argtypes = [_vp, _f32p, C.c_size_t]
    L.npsd_b200_set_mask.argtypes = [_vp, _u8p]
    L.npsd_b200_set_mask_device.argtypes = [_vp, _vp]
    L.npsd_b200_n_fluid.restype = C.c_int64
    L.npsd_b200_n_fluid.argtypes = [_vp]
    L.npsd_b200_fluid_indices.argtypes = [_vp, _i64p]
    L.npsd_b200_set_exact.argtypes = [_vp, C.c_int]
    L.npsd_b200_is_pure_neumann.argtypes = [_vp, C.POINTER(C.c_int)]
    L.npsd_b200_check_operator.argtypes = [_vp, C.c_int64, _i64p, _i64p, _f64p, C.c_int64, C.c_int]
    L.npsd_b200_precond_apply.argtypes = [_vp, _f64p, _f64p, C.c_int64]
    L.npsd_b200_psdo_solve.argtypes = [_vp, _f64p, _vp, C.POINTER(SolveCfg), _f64p, C.POINTER(Report)]
    L.npsd_b200_psdo_solve_n.argtypes = [_vp, _f64p, C.c_int64, _vp, C.POINTER(SolveCfg), _f64p, C.POINTER(Report)]
    L.npsd_b200_psdo_solve_device.argtypes = [_vp, _vp, _vp, C.POINTER(SolveCfg), _vp, C.POINTER(Report)]
    L.npsd_b200_spmv.argtypes = [_vp, _f64p, _f64p, C.c_int64]
    L.npsd_b200_net_apply.argtypes = [_vp, _f32p, _f32p]
    L.npsd_b200_level_image.argtypes = [_vp, C.c_int, _f32p]
    L.npsd_b200_linear_coeffs.argtypes = [_vp, _f32p, _f32p]
    L.npsd_b200_mixed_counts.argtypes = [_vp, _i64p]
    L.npsd_b200_param_count.restype = C.c_size_t
    L.npsd_b200_param_count.argtypes = [C.c_int, C.c_int]
    L.npsd_b200_init_params.argtypes = [C.c_int, C.c_int, C.c_uint64, _f32p]
    L.npsd_b200_identity_params.argtypes = [C.c_int, C.c_int, _f32p]
    L.npsd_b200_rhs_normal.argtypes = [C.c_uint64, C.c_int64, _f64p]
    L.npsd_b200_device_alloc.argtypes = [_vp, C.c_size_t, C.POINTER(_vp)]
    L.npsd_b200_device_free.argtypes = [_vp, _vp]
    L.npsd_b200_host_alloc.argtypes = [_vp, C.c_size_t, C.POINTER(_vp)]
    L.npsd_b200_host_free.argtypes = [_vp, _vp]
    L.npsd_b200_memcpy.argtypes = [_vp, _vp, _vp, C.c_size_t]
    L.npsd_b200_synchronize.argtypes = [_vp]
    L.npsd_b200_last_solve_ms.restype = C.c_double
    L.npsd_b200_last_solve_ms.argtypes = [_vp]
    L.npsd_b200_last_solve_launches.restype = C.c_int64
    L.npsd_b200_last_solve_launches.argtypes = [_vp]
    L.npsd_b200_launch_count.restype = C.c_int64
    L.npsd_b200_launch_count.argtypes = [_vp]
    L.npsd_b200_event_record.argtypes = [_vp, C.c_int]
    L.npsd_b200_event_elapsed_ms.restype = C.c_double
    L.npsd_b200_event_elapsed_ms.argtypes = [_vp, C.c_int, C.c_int]
    L.npsd_b200_profile_iterations.argtypes = [_vp, _vp, C.POINTER(SolveCfg), C.c_int, _f64p, C.POINTER(C.c_int),
                                               C.c_char_p, C.c_int]
    _lib = L
    return L
