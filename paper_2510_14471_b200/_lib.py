"""ctypes binding of the in-tree CUDA library libglsgpu.so (the C-ABI of include/glsgpu.h).

There is no CPU fallback: if the library is missing or no CUDA device is present, every entry point
raises.  The library is loaded from this package directory only (it travels with the repo snapshot).
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libglsgpu.so")

_P = C.POINTER(C.c_double)
_PI64 = C.POINTER(C.c_int64)


class PcgConfigC(C.Structure):
    _fields_ = [("tol_rel", C.c_double), ("max_iter", C.c_int64), ("breakdown_tol", C.c_double),
                ("stagnation_window", C.c_int64), ("growth_tol", C.c_double), ("growth_window", C.c_int64),
                ("record_z_every", C.c_int64), ("diag_every", C.c_int32), ("xv_mode", C.c_int32),
                ("graph_chunk", C.c_int32), ("kernel_timing", C.c_int32),
                ("kron_fma", C.c_int32), ("sw_mode", C.c_int32),
                ("fused_c", C.c_int32)]


class TraceRowC(C.Structure):
    _fields_ = [("iter", C.c_int64), ("c", C.c_double), ("aug_residual_norm", C.c_double),
                ("dual_feas_norm", C.c_double), ("rmse", C.c_double), ("elapsed_ns", C.c_int64)]


class ResultC(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("termination", C.c_int32), ("w1_projected", C.c_int32),
                ("breakdown_iteration", C.c_int64), ("residual_seminorm", C.c_double), ("n_rows", C.c_int64),
                ("sigma_scale", C.c_double), ("solve_ms", C.c_double)]


class CountersC(C.Structure):
    _fields_ = [("factorizations", C.c_uint64), ("factor_multiplies", C.c_uint64), ("pi_applies", C.c_uint64),
                ("xstar_t_applies", C.c_uint64), ("xstar_applies", C.c_uint64), ("apply_multiplies", C.c_uint64)]


class KernelStatC(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", C.c_int64), ("total_ms", C.c_double),
                ("bytes_per_launch", C.c_double)]


# every symbol include/glsgpu.h declares (tests check the export table)
EXPORTS = [
    "glsgpu_device_count", "glsgpu_last_error_message", "glsgpu_version", "glsgpu_sur_create",
    "glsgpu_sur_create_device", "glsgpu_sur_refactor", "glsgpu_sur_destroy", "glsgpu_sur_dims", "glsgpu_sur_stream",
    "glsgpu_apply_pi", "glsgpu_apply_xstar_t", "glsgpu_apply_xstar", "glsgpu_sigma_apply",
    "glsgpu_operator_norm_probe", "glsgpu_counters", "glsgpu_reset_apply_counters", "glsgpu_sur_solve",
    "glsgpu_default_config", "glsgpu_kernel_stats", "glsgpu_launch_count", "glsgpu_get_factors", "glsgpu_synth_normal",
    "glsgpu_synth_response", "glsgpu_nccl_unique_id", "glsgpu_sur_create_sharded", "glsgpu_sur_shard",
    "glsgpu_mvrglm_create", "glsgpu_mv_reduce", "glsgpu_model_dims", "glsgpu_sur_reduce", "glsgpu_pcg_ne", "glsgpu_sur_update",
    "glsgpu_sur_stage", "glsgpu_sur_update_staged", "glsgpu_sur_create_sharded_host", "glsgpu_local_group_create",
    "glsgpu_local_group_destroy", "glsgpu_sur_create_sharded_local", "glsgpu_factor_info",
]

_lib = None


def load() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2510_14471_b200.build` "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    H = C.c_void_p
    L.glsgpu_device_count.argtypes = [C.POINTER(C.c_int)]
    L.glsgpu_last_error_message.restype = C.c_char_p
    L.glsgpu_version.restype = C.c_char_p
    L.glsgpu_sur_create.argtypes = [C.c_int, C.c_int64, _PI64, _P, _P, _P, _P, C.c_int, C.POINTER(H),
                                    C.POINTER(C.c_int)]
    L.glsgpu_sur_create_device.argtypes = [C.c_int, C.c_int64, _PI64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                           _P, _P, C.c_int, C.POINTER(H), C.POINTER(C.c_int)]
    L.glsgpu_sur_refactor.argtypes = [H, C.POINTER(C.c_int)]
    L.glsgpu_sur_update.argtypes = [H, _P, _P, C.POINTER(C.c_int)]
    L.glsgpu_sur_stage.argtypes = [H, C.c_void_p, C.c_void_p]
    L.glsgpu_sur_update_staged.argtypes = [H, C.POINTER(C.c_int)]
    L.glsgpu_sur_create_sharded_host.argtypes = [C.c_int, C.c_int64, C.c_int64, _PI64, C.c_void_p, C.c_void_p, _P, _P,
                                                 C.c_int, C.c_void_p, C.c_int, C.c_int, C.POINTER(H),
                                                 C.POINTER(C.c_int)]
    L.glsgpu_local_group_create.argtypes = [C.c_int, C.c_int, C.POINTER(H)]
    L.glsgpu_local_group_destroy.argtypes = [H]
    L.glsgpu_sur_create_sharded_local.argtypes = [C.c_int, C.c_int64, C.c_int64, _PI64, C.c_void_p, C.c_int64,
                                                  C.c_void_p, C.c_int64, _P, _P, H, C.c_int, C.POINTER(H),
                                                  C.POINTER(C.c_int)]
    L.glsgpu_sur_destroy.argtypes = [H]
    L.glsgpu_sur_dims.argtypes = [H, C.POINTER(C.c_int), _PI64, _PI64]
    L.glsgpu_sur_stream.argtypes = [H]
    L.glsgpu_sur_stream.restype = C.c_void_p
    for f in ("glsgpu_apply_pi", "glsgpu_apply_xstar_t", "glsgpu_apply_xstar", "glsgpu_sigma_apply"):
        getattr(L, f).argtypes = [H, _P, _P]
    L.glsgpu_operator_norm_probe.argtypes = [H, C.c_int64, _P]
    L.glsgpu_counters.argtypes = [H, C.POINTER(CountersC)]
    L.glsgpu_reset_apply_counters.argtypes = [H]
    L.glsgpu_sur_solve.argtypes = [H, C.POINTER(PcgConfigC), _P, _P, _P, _P, _P, C.POINTER(TraceRowC), C.c_int64,
                                   C.POINTER(ResultC)]
    L.glsgpu_default_config.argtypes = [C.POINTER(PcgConfigC)]
    L.glsgpu_default_config.restype = None
    L.glsgpu_kernel_stats.argtypes = [H, C.POINTER(KernelStatC), C.c_int]
    L.glsgpu_launch_count.argtypes = [H, _PI64]
    L.glsgpu_get_factors.argtypes = [H, _P, _P]
    L.glsgpu_factor_info.argtypes = [H, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    L.glsgpu_synth_normal.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_uint64,
                                      C.c_uint64, C.c_int]
    L.glsgpu_synth_response.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int64, _PI64, C.c_void_p, C.c_int64, _P, _P,
                                        C.c_uint64, C.c_void_p, C.c_int64, C.c_int]
    L.glsgpu_nccl_unique_id.argtypes = [C.c_void_p]
    L.glsgpu_sur_create_sharded.argtypes = [C.c_int, C.c_int64, C.c_int64, _PI64, C.c_void_p, C.c_int64, C.c_void_p,
                                            C.c_int64, _P, _P, C.c_int, C.c_void_p, C.c_int, C.c_int, C.POINTER(H),
                                            C.POINTER(C.c_int)]
    L.glsgpu_sur_shard.argtypes = [H, C.POINTER(C.c_int), C.POINTER(C.c_int), _PI64]
    L.glsgpu_mvrglm_create.argtypes = [C.c_int, C.c_int64, C.c_int64, _P, _P, _P, _PI64, _PI64, _P, _P, C.c_int,
                                       C.POINTER(H), C.POINTER(C.c_int)]
    L.glsgpu_mv_reduce.argtypes = [C.c_int, C.c_int64, C.c_int64, _P, _P, _P, _P, C.c_int]
    L.glsgpu_model_dims.argtypes = [H, _PI64, _PI64]
    L.glsgpu_pcg_ne.argtypes = [H, C.POINTER(PcgConfigC), _P, _P, _P, C.POINTER(TraceRowC), C.c_int64,
                                C.POINTER(ResultC)]
    L.glsgpu_sur_reduce.argtypes = [C.c_int, C.c_int64, _PI64, _P, _P, C.c_double, C.c_int, _PI64, _P, _P, _P]
    _lib = L
    return L
