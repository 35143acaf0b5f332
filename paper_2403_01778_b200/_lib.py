"""ctypes binding of librank1_b200.so (the C-ABI declared in include/rank1_b200.h).

Loading fails loudly when the library is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
# R1_LIB_PATH: development A/B runs against another build of this library
LIB_PATH = os.environ.get("R1_LIB_PATH", os.path.join(PKG, "librank1_b200.so"))

_dp = ctypes.POINTER(ctypes.c_double)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_vp = ctypes.c_void_p

R1_OK = 0
R1_ERR_INVALID_ARGUMENT = 1
R1_ERR_RUNTIME = 2
R1_ERR_CUDA = 3
R1_ERR_NO_DEVICE = 4
R1_ERR_INTERNAL = 5


class Rank1Error(Exception):
    """Base of all errors raised through the C-ABI."""


class InvalidArgument(Rank1Error, ValueError):
    """std::invalid_argument in the reference."""


class Rank1RuntimeError(Rank1Error, RuntimeError):
    """std::runtime_error in the reference."""


class DeviceError(Rank1Error, RuntimeError):
    """CUDA failure or no usable B200 (there is no CPU fallback)."""


class SolveOptionsC(ctypes.Structure):
    _fields_ = [("tol", ctypes.c_double), ("max_iters", ctypes.c_int32),
                ("init", ctypes.c_int32), ("seed", ctypes.c_uint64),
                ("init_factors", _dp), ("determinism", ctypes.c_int32),
                ("rqi_accept_rule", ctypes.c_int32), ("stop_rule", ctypes.c_int32),
                ("threads", ctypes.c_int32), ("record_kkt", ctypes.c_int32),
                ("asvd_disjoint_pairs", ctypes.c_int32),
                ("reuse_intermediates", ctypes.c_int32), ("scf_lambda_rtol", ctypes.c_double),
                ("scf_angle_tol", ctypes.c_double)]


class IterationRecordC(ctypes.Structure):
    _fields_ = [("lambda_", ctypes.c_double), ("stop_value", ctypes.c_double),
                ("eq11_value", ctypes.c_double), ("kkt_max_residual", ctypes.c_double),
                ("rqi_accepted", ctypes.c_int32), ("n_sweeps", ctypes.c_int32),
                ("lambda_pre_rqi", ctypes.c_double), ("t_build_j", ctypes.c_double),
                ("t_eig", ctypes.c_double), ("t_other", ctypes.c_double),
                ("factor_change", ctypes.c_double)]


class SolveReportC(ctypes.Structure):
    _fields_ = [("lambda_", ctypes.c_double), ("factors", _dp), ("converged", ctypes.c_int32),
                ("iterations", ctypes.c_int32), ("lambda0", ctypes.c_double),
                ("restarted", ctypes.c_int32), ("final_x", _dp),
                ("trace", ctypes.POINTER(IterationRecordC)), ("total_sweeps", ctypes.c_int32),
                ("t_total", ctypes.c_double)]


class GreedyReportC(ctypes.Structure):
    _fields_ = [("completed", ctypes.c_int32), ("terms", ctypes.c_int32), ("lambdas", _dp),
                ("factors", _dp), ("residual_ratios", _dp),
                ("solves", ctypes.POINTER(SolveReportC)), ("failure", ctypes.c_char * 256)]


# name -> (restype, argtypes): every symbol include/rank1_b200.h declares.
SIGNATURES = {
    "r1_abi_version": (ctypes.c_int, []),
    "r1_last_error": (ctypes.c_char_p, []),
    "r1_device_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    "r1_solve_options_default": (None, [ctypes.POINTER(SolveOptionsC)]),
    "r1_context_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_vp)]),
    "r1_context_destroy": (ctypes.c_int, [_vp]),
    "r1_context_set_stream": (ctypes.c_int, [_vp, _vp]),
    "r1_context_synchronize": (ctypes.c_int, [_vp]),
    "r1_context_launch_count": (ctypes.c_int, [_vp, _u64p]),
    "r1_tensor_from_host": (ctypes.c_int, [_vp, _dp, _u64p, ctypes.c_int, ctypes.POINTER(_vp)]),
    "r1_tensor_create": (ctypes.c_int, [_vp, _u64p, ctypes.c_int, ctypes.POINTER(_vp)]),
    "r1_tensor_wrap_device": (ctypes.c_int, [_vp, _vp, _u64p, ctypes.c_int, ctypes.POINTER(_vp)]),
    "r1_host_register": (ctypes.c_int, [_vp, ctypes.c_uint64]),
    "r1_host_unregister": (ctypes.c_int, [_vp]),
    "r1_tensor_copy_from_host": (ctypes.c_int, [_vp, _vp, _dp]),
    "r1_tensor_copy_to_host": (ctypes.c_int, [_vp, _vp, _dp]),
    "r1_tensor_frobenius": (ctypes.c_int, [_vp, _vp, _dp]),
    "r1_host_frobenius": (ctypes.c_int, [_vp, _dp, _u64p, ctypes.c_int, _dp]),
    "r1_tensor_destroy": (ctypes.c_int, [_vp]),
    "r1_tensor_device_ptr": (_vp, [_vp]),
    "r1_blocks_numel": (ctypes.c_uint64, [_u64p, ctypes.c_int]),
    "r1_build_j_device": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "r1_build_j": (ctypes.c_int, [_vp, _dp, _vp, _u64p, ctypes.c_int, _dp, _dp]),
    "r1_build_block": (ctypes.c_int, [_vp, _dp, _vp, _u64p, ctypes.c_int, _dp, ctypes.c_int,
                                      ctypes.c_int, _dp]),
    "r1_block_matvec_device": (ctypes.c_int, [_vp, _u64p, ctypes.c_int, _vp, _vp, _vp]),
    "r1_contract_leaving_all": (ctypes.c_int, [_vp, _dp, _vp, _u64p, ctypes.c_int, _dp, _dp]),
    "r1_block_matvec": (ctypes.c_int, [_vp, _u64p, ctypes.c_int, _dp, _dp, _dp]),
    "r1_block_dense": (ctypes.c_int, [_vp, _u64p, ctypes.c_int, _dp, _dp]),
    "r1_block_frobenius": (ctypes.c_int, [_vp, _u64p, ctypes.c_int, _dp, _dp]),
    "r1_scf_stopping_value": (ctypes.c_int, [_vp, _u64p, ctypes.c_int, _dp, _dp, ctypes.c_double,
                                             _dp]),
    "r1_kkt_from_blocks": (ctypes.c_int, [_vp, _u64p, ctypes.c_int, _dp, _dp, _dp]),
    "r1_kkt_report": (ctypes.c_int, [_vp, _dp, _vp, _u64p, ctypes.c_int, _dp, _dp]),
    "r1_eig_blocks_device": (ctypes.c_int, [_vp, _u64p, ctypes.c_int, _vp, _vp, _vp, _vp]),
    "r1_largest_magnitude_eigenpair": (ctypes.c_int, [_vp, ctypes.c_int64, _dp, _dp, _dp]),
    "r1_rayleigh_quotient_step": (ctypes.c_int, [_vp, ctypes.c_int64, _dp, _dp, _dp,
                                                 ctypes.POINTER(ctypes.c_int)]),
    "r1_generate_config": (ctypes.c_int, [_vp, _vp, ctypes.c_int, ctypes.c_uint64, _u64p,
                                          ctypes.c_int, ctypes.c_uint64]),
    "r1_rqi_blocks_device": (ctypes.c_int, [_vp, _u64p, ctypes.c_int, _vp, _vp, _vp,
                                            ctypes.POINTER(ctypes.c_int)]),
    "r1_generate": (ctypes.c_int, [_vp, _vp, ctypes.c_char_p, ctypes.c_uint64]),
    "r1_solve": (ctypes.c_int, [_vp, ctypes.c_char_p, _vp, ctypes.POINTER(SolveOptionsC),
                                ctypes.POINTER(SolveReportC)]),
    "r1_solve_host": (ctypes.c_int, [_vp, ctypes.c_char_p, _dp, _u64p, ctypes.c_int,
                                     ctypes.POINTER(SolveOptionsC), ctypes.POINTER(SolveReportC)]),
    "r1_comm_unique_id": (ctypes.c_int, [_vp]),
    "r1_comm_init": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _vp, ctypes.POINTER(_vp)]),
    "r1_comm_init_all": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                        ctypes.POINTER(_vp), ctypes.POINTER(_vp)]),
    "r1_comm_destroy": (ctypes.c_int, [_vp]),
    "r1_comm_info": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]),
    "r1_slab_bounds": (ctypes.c_int, [ctypes.c_uint64, ctypes.c_int, ctypes.c_int, _u64p, _u64p]),
    "r1_build_j_sharded": (ctypes.c_int, [_vp, _vp, _u64p, ctypes.c_int, _vp, _vp, _vp]),
    "r1_solve_sharded": (ctypes.c_int, [_vp, ctypes.c_char_p, _vp, _u64p, ctypes.c_int,
                                        ctypes.POINTER(SolveOptionsC), ctypes.POINTER(SolveReportC)]),
    "r1_greedy_rank_r": (ctypes.c_int, [_vp, _vp, ctypes.c_uint64, ctypes.c_char_p,
                                        ctypes.POINTER(SolveOptionsC), ctypes.POINTER(GreedyReportC)]),
    "r1_rank_one_subtract": (ctypes.c_int, [_vp, _vp, ctypes.c_double, _dp, _dp]),
    "r1_sym_eig_full": (ctypes.c_int, [_vp, ctypes.c_int64, _dp, _dp, _dp]),
    "r1_ldlt_factor": (ctypes.c_int, [_vp, ctypes.c_int64, _dp, _dp, ctypes.POINTER(ctypes.c_int),
                                      ctypes.POINTER(ctypes.c_int)]),
    "r1_ldlt_solve": (ctypes.c_int, [_vp, ctypes.c_int64, _dp, ctypes.POINTER(ctypes.c_int), _dp,
                                     _dp]),
    "r1_ldlt_diag_condition": (ctypes.c_int, [_vp, ctypes.c_int64, _dp, _dp,
                                              ctypes.POINTER(ctypes.c_int), ctypes.c_int, _dp]),
    "r1_matricize": (ctypes.c_int, [_vp, _dp, _u64p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp]),
    "r1_ttvc": (ctypes.c_int, [_vp, _dp, _u64p, ctypes.c_int, _dp, ctypes.POINTER(ctypes.c_int),
                               ctypes.c_int, ctypes.c_int, _dp, _dp]),
    "r1_rank_one_expand": (ctypes.c_int, [_vp, ctypes.c_double, _dp, _u64p, ctypes.c_int, _dp]),
    "r1_residual_norm": (ctypes.c_int, [_vp, _dp, _u64p, ctypes.c_int, ctypes.c_double, _dp,
                                        ctypes.c_uint64, _dp]),
    "r1_tensor_read_dt1": (ctypes.c_int, [_vp, ctypes.c_char_p, ctypes.POINTER(_vp)]),
    "r1_tensor_write_dt1": (ctypes.c_int, [_vp, _vp, ctypes.c_char_p]),
}

# Diagnostics not in the public header (tests / bench only).
EXTRA_SIGNATURES = {
    "r1x_set_sweep_trace": (ctypes.c_int, [_vp, _vp]),
    "r1x_time_kernels": (ctypes.c_int, [_vp, ctypes.c_int]),
    "r1x_kernel_time": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_double),
                                       ctypes.POINTER(ctypes.c_uint64)]),
    "r1x_eig_blocks_info": (ctypes.c_int, [_vp, _u64p, ctypes.c_int, _dp, _dp, _dp,
                                           ctypes.POINTER(ctypes.c_int), _dp]),
    "r1x_sweep_plan_info": (ctypes.c_int, [_vp, _u64p, ctypes.c_int,
                                           ctypes.POINTER(ctypes.c_int64)]),
    "r1x_exchange_plan": (ctypes.c_int, [_u64p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.POINTER(ctypes.c_int64), ctypes.c_int]),
    "r1x_solver_graph_mode": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_int)]),
    "r1x_eig_dense_lanczos": (ctypes.c_int, [_vp, ctypes.c_int64, _dp, _dp, _dp]),
    "r1x_ldlt": (ctypes.c_int, [_vp, ctypes.c_int64, _dp, ctypes.POINTER(ctypes.c_int), _dp, _dp,
                                ctypes.POINTER(ctypes.c_int), _dp]),
    "r1x_ldlt_time": (ctypes.c_int, [_vp, ctypes.c_int64, _dp, ctypes.c_int, _dp]),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError(f"{LIB_PATH} is not built (run paper_2403_01778_b200/build.py); "
                              "there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in {**SIGNATURES, **EXTRA_SIGNATURES}.items():
            fn = getattr(L, name, None)
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == R1_OK:
        return
    msg = (lib().r1_last_error() or b"").decode(errors="replace")
    if rc == R1_ERR_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if rc == R1_ERR_RUNTIME:
        raise Rank1RuntimeError(msg)
    if rc in (R1_ERR_CUDA, R1_ERR_NO_DEVICE):
        raise DeviceError(msg)
    raise Rank1Error(msg)


def dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_dp)


def dims_arr(dims) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(dims, dtype=np.uint64))


def u64p(a: np.ndarray):
    return a.ctypes.data_as(_u64p)
