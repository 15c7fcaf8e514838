"""ctypes binding of libsap_gpu.so (the C ABI declared in include/sap_gpu.h).

There is no fallback: if the shared library is missing or cannot be loaded
this module raises, so nothing can silently run the hot path elsewhere.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SAP_GPU_LIB", os.path.join(_HERE, "libsap_gpu.so"))  # tools: A/B builds


class sap_options(C.Structure):
    _fields_ = [("p", C.c_int), ("precond", C.c_int), ("boost_eps", C.c_double), ("method", C.c_int),
                ("ell", C.c_int), ("rel_tol", C.c_double), ("abs_tol", C.c_double), ("max_iterations", C.c_int),
                ("mixed_precision", C.c_int), ("caller_asserts_spd", C.c_int), ("device", C.c_int),
                ("triangle_solve", C.c_int), ("lu_kernel", C.c_int), ("tip_solve", C.c_int)]


class sap_report(C.Structure):
    _fields_ = [("t_lu", C.c_double), ("t_bc", C.c_double), ("t_spk", C.c_double), ("t_lurdcd", C.c_double),
                ("t_kry", C.c_double), ("t_dtransf", C.c_double), ("n", C.c_int), ("k", C.c_int),
                ("partitions", C.c_int), ("total_boosts", C.c_int), ("total_boosts_ul", C.c_int),
                ("total_rbar_boosts", C.c_int), ("kernel_launches", C.c_longlong),
                ("t_factor_kernel", C.c_double), ("factor_flops", C.c_double), ("chunk_condition", C.c_double),
                ("sweep_substitution", C.c_int), ("t_drop", C.c_double), ("t_asmbl", C.c_double),
                ("krylov_host_syncs", C.c_longlong), ("ul_tip_sweeps", C.c_int)]


class sap_solve_stats(C.Structure):
    _fields_ = [("iterations", C.c_double), ("converged", C.c_int), ("final_relative_residual", C.c_double),
                ("failure", C.c_int), ("history_len", C.c_int), ("history", C.POINTER(C.c_double)),
                ("history_capacity", C.c_int)]


ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int)
EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int,
                          C.c_void_p, C.c_int)


class sap_comm(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("rank", C.c_int), ("world", C.c_int), ("allreduce_sum", ALLREDUCE_FN),
                ("exchange", EXCHANGE_FN)]


# Every symbol include/sap_gpu.h declares, with its ctypes signature.
_vp = C.c_void_p
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
SIGNATURES = {
    "sap_options_default": (None, [C.POINTER(sap_options)]),
    "sap_max_feasible_partitions": (C.c_int, [C.c_int, C.c_int]),
    "sap_partition_layout": (C.c_int, [C.c_int, C.c_int, C.c_int, _ip, _ip]),
    "sap_last_error": (C.c_char_p, []),
    "sap_status_string": (C.c_char_p, [C.c_int]),
    "sap_version": (C.c_char_p, []),
    "sap_random_banded": (C.c_int, [C.c_int, C.c_int, C.c_double, C.c_uint, _vp, _vp]),
    "sap_create": (C.c_int, [C.POINTER(sap_options), C.POINTER(_vp)]),
    "sap_destroy": (None, [_vp]),
    "sap_set_stream": (C.c_int, [_vp, _vp]),
    "sap_synchronize": (C.c_int, [_vp]),
    "sap_setup_banded": (C.c_int, [_vp, C.c_int, C.c_int, _vp, C.c_int]),
    "sap_set_operator_csr": (C.c_int, [_vp, C.c_int, C.c_int, _vp, _vp, _vp, C.c_int]),
    "sap_setup_banded_from_csr": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, C.c_int]),
    "sap_apply_preconditioner": (C.c_int, [_vp, _vp, _vp, C.c_int]),
    "sap_apply_operator": (C.c_int, [_vp, _vp, _vp, C.c_int]),
    "sap_solve": (C.c_int, [_vp, _vp, _vp, C.c_int, C.POINTER(sap_solve_stats)]),
    "sap_get_report": (C.c_int, [_vp, C.POINTER(sap_report)]),
    "sap_get_factor": (C.c_int, [_vp, C.c_int, C.c_int, _vp, _ip, _dp]),
    "sap_get_spike": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp, _vp, _vp, _ip]),
    "sap_setup_from_csr_drop": (C.c_int, [_vp, C.c_int, C.c_int, _vp, _vp, _vp, C.c_double, C.c_int, _ip]),
    "sap_set_third_stage": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp, C.c_int]),
    "sap_get_full_spike": (C.c_int, [_vp, C.c_int, _vp, _vp]),
    "sap_rank_rows": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _ip, _ip]),
    "sap_create_distributed": (C.c_int, [C.POINTER(sap_options), C.POINTER(sap_comm), C.POINTER(_vp)]),
    "sap_nccl_get_unique_id": (C.c_int, [_vp]),
    "sap_create_distributed_nccl": (C.c_int, [C.POINTER(sap_options), _vp, C.c_int, C.c_int, C.POINTER(_vp)]),
    "sap_setup_banded_dist": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.c_int, _vp, C.c_int]),
}

_lib = None


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libsap_gpu.so not built at {LIB_PATH}; run `python -m paper_1509_07919_b200.build` "
                              "(there is no CPU fallback for the SaP hot path)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib
