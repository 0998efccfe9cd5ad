"""ctypes binding of libequil_b200.so (the C ABI in include/equil_b200.h).

The product path has no fallback: if the shared library is missing or fails to
load, importing the API raises.  Build it with
``python -m paper_1602_06621_b200.build``.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EQUIL_LIB") or os.path.join(HERE, "libequil_b200.so")

EQUIL_OK, EQUIL_EINVAL, EQUIL_ERUNTIME, EQUIL_ECUDA, EQUIL_ENCCL, EQUIL_ENOMEM = range(6)

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_u32p = C.POINTER(C.c_uint32)
_ip = C.POINTER(C.c_int)


class Params(C.Structure):
    _fields_ = [("alpha", C.c_double), ("beta", C.c_double), ("gamma", C.c_double),
                ("max_log_scale", C.c_double), ("iterations", C.c_int),
                ("seed", C.c_uint64)]


class DeviceCfg(C.Structure):
    _fields_ = [("device", C.c_int), ("rank", C.c_int), ("world_size", C.c_int),
                ("nccl_id", C.c_void_p)]


class DiagCfg(C.Structure):
    _fields_ = [("stride", C.c_int), ("want_objective", C.c_int), ("want_rms", C.c_int)]


class ScalingOut(C.Structure):
    _fields_ = [("u", _dp), ("v", _dp), ("d", _dp), ("e", _dp),
                ("outputs_on_device", C.c_int), ("alpha", C.c_double),
                ("beta", C.c_double), ("box_feasible", C.c_int),
                ("iterate_bound_ok", C.c_int), ("apply_count", C.c_longlong),
                ("adjoint_count", C.c_longlong), ("hist_iter", _ip),
                ("hist_objective", _dp), ("hist_rms", _dp), ("hist_cap", C.c_int),
                ("hist_len", C.c_int)]


class LsqrOut(C.Structure):
    _fields_ = [("x", _dp), ("residual_history", _dp), ("residual_cap", C.c_int),
                ("hist_len", C.c_int), ("iterations", C.c_int),
                ("equil_iterations", C.c_int), ("reached_tol", C.c_int),
                ("breakdown", C.c_int), ("apply_count", C.c_longlong),
                ("adjoint_count", C.c_longlong)]


class CcpOptions(C.Structure):
    _fields_ = [("max_iters", C.c_int), ("tau", C.c_double), ("sigma", C.c_double),
                ("theta", C.c_double), ("p_star", C.c_double), ("gap_tol", C.c_double)]


class CcpOut(C.Structure):
    _fields_ = [("x", _dp), ("objective_history", _dp), ("gap_history", _dp),
                ("hist_cap", C.c_int), ("hist_len", C.c_int), ("gap_len", C.c_int),
                ("tau", C.c_double), ("sigma", C.c_double), ("theta", C.c_double),
                ("iterations", C.c_int), ("equil_iterations", C.c_int),
                ("reached_tol", C.c_int), ("apply_count", C.c_longlong),
                ("adjoint_count", C.c_longlong)]


# matrix-free operator (equil_device_operator): apply(ctx, in, out, stream)
DeviceApplyFn = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p)


class DeviceOperator(C.Structure):
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("apply", DeviceApplyFn),
                ("apply_adjoint", DeviceApplyFn), ("ctx", C.c_void_p), ("device", C.c_int)]


# every exported symbol of include/equil_b200.h with (restype, argtypes)
SIGNATURES = {
    "equil_params_default": (None, [C.POINTER(Params)]),
    "equil_resolve_targets": (C.c_int, [C.POINTER(Params), C.c_int64, C.c_int64, _dp, _dp]),
    "equil_validate_params": (C.c_int, [C.POINTER(Params)]),
    "equil_matrix_create_csr": (C.c_int, [C.c_int64, C.c_int64, _i64p, _i32p, _dp,
                                          C.POINTER(DeviceCfg), C.POINTER(C.c_void_p)]),
    "equil_matrix_create_coo": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, _i64p, _i64p, _dp,
                                          C.POINTER(DeviceCfg), C.POINTER(C.c_void_p)]),
    "equil_matrix_create_dense": (C.c_int, [C.c_int64, C.c_int64, _dp,
                                            C.POINTER(DeviceCfg), C.POINTER(C.c_void_p)]),
    "equil_matrix_destroy": (None, [C.c_void_p]),
    "equil_matrix_shape": (C.c_int, [C.c_void_p, _i64p, _i64p, _i64p]),
    "equil_matrix_stream": (C.c_void_p, [C.c_void_p]),
    "equil_last_loop_ms": (C.c_double, [C.c_void_p, _ip]),
    "equil_exchange_mode": (C.c_int, [C.c_void_p]),
    "equil_sweep_active": (C.c_int, [C.c_void_p]),
    "equil_kernel_launches": (C.c_longlong, []),
    "equil_build_flags": (C.c_int, []),
    "equil_apply": (C.c_int, [C.c_void_p, _dp, _dp, C.c_int]),
    "equil_apply_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]),
    "equil_sgd_equilibrate_operator": (C.c_int, [C.POINTER(DeviceOperator), C.POINTER(Params),
                                                 C.POINTER(ScalingOut)]),
    "equil_lsqr_operator": (C.c_int, [C.POINTER(DeviceOperator), _dp, C.POINTER(Params),
                                      C.c_int, C.c_double, C.POINTER(LsqrOut)]),
    "equil_sgd_equilibrate": (C.c_int, [C.c_void_p, C.POINTER(Params), C.POINTER(DiagCfg),
                                        C.POINTER(ScalingOut)]),
    "equil_sgd_equilibrate_targets": (C.c_int, [C.c_void_p, _dp, _dp, C.POINTER(Params),
                                                C.POINTER(DiagCfg), C.POINTER(ScalingOut)]),
    "equil_sgd_equilibrate_symmetric": (C.c_int, [C.c_void_p, C.POINTER(Params),
                                                  C.POINTER(DiagCfg), C.POINTER(ScalingOut)]),
    "equil_sgd_equilibrate_block": (C.c_int, [C.c_void_p, _i64p, _i64p, C.c_int64, C.c_int64,
                                              C.POINTER(Params), C.POINTER(DiagCfg),
                                              C.POINTER(ScalingOut)]),
    "equil_ccp_lasso": (C.c_int, [C.c_void_p, _dp, C.c_double, C.POINTER(CcpOptions),
                                  C.POINTER(CcpOut)]),
    "equil_ccp_lasso_preconditioned": (C.c_int, [C.c_void_p, _dp, C.c_double,
                                                 C.POINTER(Params), C.POINTER(CcpOptions),
                                                 C.POINTER(CcpOut)]),
    "equil_spectral_norm": (C.c_int, [C.c_void_p, C.c_int, C.c_double, C.c_uint64, _dp]),
    "equil_lasso_objective": (C.c_int, [C.c_void_p, _dp, C.c_double, _dp, _dp]),
    "equil_matrix_read_matrix_market": (C.c_int, [C.c_char_p, C.POINTER(DeviceCfg),
                                                  C.POINTER(C.c_void_p)]),
    "equil_matrix_write_matrix_market": (C.c_int, [C.c_void_p, C.c_char_p]),
    "equil_matrix_save_binary": (C.c_int, [C.c_void_p, C.c_char_p]),
    "equil_matrix_load_binary": (C.c_int, [C.c_char_p, C.POINTER(DeviceCfg),
                                           C.POINTER(C.c_void_p)]),
    "equil_matrix_export_csr": (C.c_int, [C.c_void_p, _i64p, _i32p, _dp]),
    "equil_matrix_export_dense": (C.c_int, [C.c_void_p, _dp]),
    "equil_matrix_is_dense": (C.c_int, [C.c_void_p]),
    "equil_mm_parse": (C.c_int, [C.c_char_p, _i64p, _i64p, _i64p, C.POINTER(C.c_int),
                                 C.POINTER(C.c_void_p)]),
    "equil_mm_fetch": (C.c_int, [C.c_void_p, _i64p, _i64p, _dp, _i64p]),
    "equil_mm_free": (None, [C.c_void_p]),
    "equil_mm_write_csr": (C.c_int, [C.c_char_p, C.c_int64, C.c_int64, _i64p, _i32p, _dp]),
    "equil_mm_write_dense": (C.c_int, [C.c_char_p, C.c_int64, C.c_int64, _dp]),
    "equil_objective": (C.c_int, [C.c_void_p, _dp, _dp, C.POINTER(Params), _dp]),
    "equil_objective_weighted": (C.c_int, [C.c_void_p, _dp, _dp, _dp, _dp, C.c_double, _dp]),
    "equil_gradient": (C.c_int, [C.c_void_p, _dp, _dp, C.POINTER(Params), _dp, _dp]),
    "equil_gradient_weighted": (C.c_int, [C.c_void_p, _dp, _dp, _dp, _dp, C.c_double, _dp,
                                          _dp]),
    "equil_stochastic_gradient_estimate": (C.c_int, [C.c_void_p, _dp, _dp, C.POINTER(Params),
                                                     C.c_uint64, C.c_uint64, C.c_uint64, _dp,
                                                     _dp]),
    "equil_rms_error": (C.c_int, [C.c_void_p, _dp, _dp, C.c_double, C.c_double, _dp]),
    "equil_project_box": (C.c_int, [_dp, C.c_int64, C.c_double, _dp]),
    "equil_lsqr": (C.c_int, [C.c_void_p, _dp, C.c_int, C.c_double, C.POINTER(LsqrOut)]),
    "equil_lsqr_preconditioned": (C.c_int, [C.c_void_p, _dp, C.POINTER(Params), C.c_int,
                                            C.c_double, C.POINTER(LsqrOut)]),
    "equil_sgd_equilibrate_csr": (C.c_int, [C.c_int64, C.c_int64, _i64p, _i32p, _dp,
                                            C.POINTER(Params), C.POINTER(DeviceCfg),
                                            C.POINTER(ScalingOut)]),
    "equil_sign_bits": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, _u32p,
                                  C.c_int]),
    "equil_export_transpose": (C.c_int, [C.c_void_p, _i64p, _i32p, _dp]),
    "equil_det_exp_device": (C.c_int, [_dp, _dp, C.c_int64, C.c_int]),
    "equil_det_exp_host": (C.c_double, [C.c_double]),
    "equil_canon_sumsq_device": (C.c_int, [_dp, C.c_int64, _dp, C.c_int]),
    "equil_partition_rows": (C.c_int, [_i64p, C.c_int64, C.c_int, _i64p]),
    "equil_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "equil_last_error": (C.c_char_p, []),
    "equil_version": (C.c_char_p, []),
}

_lib = None


def load() -> C.CDLL:
    """Load libequil_b200.so (raises if it is missing: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing; build it with `python -m paper_1602_06621_b200.build`")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def ptr(a, t):
    if a is None:
        return C.cast(None, t)
    return a.ctypes.data_as(t)
