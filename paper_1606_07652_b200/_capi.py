"""ctypes binding of include/blfmm_gpu.h (libblfmm_gpu.so, built in-tree).

There is no CPU fallback: if the CUDA extension is missing or cannot load,
every entry point raises.
"""
from __future__ import annotations

import ctypes as ct
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libblfmm_gpu.so")

OK, EINVAL, EDOMAIN, EACCURACY, ECUDA, ENCCL, ENOMEM, ELENGTH = range(8)
NSTAGES = 7
STAGE_NAMES = ("gather", "p2m", "m2m", "m2l_l2l", "l2p", "near", "combine")


class PlanDesc(ct.Structure):
    _fields_ = [
        ("d", ct.c_int),
        ("n", ct.c_longlong),
        ("coords", ct.POINTER(ct.c_double)),
        ("domain_lo", ct.c_double * 3),
        ("domain_hi", ct.c_double * 3),
        ("kernel_type", ct.c_int),
        ("kernel_shape", ct.c_double),
        ("sigma", ct.c_double),
        ("m_per_dim", ct.c_int),
        ("leaf_level", ct.c_int),
        ("grid_mode", ct.c_int),
        ("stencil_k", ct.c_int),
        ("nrhs", ct.c_int),
        ("device", ct.c_int),
        ("c_table", ct.POINTER(ct.c_double)),
        ("rank", ct.c_int),
        ("world", ct.c_int),
    ]


class Stats(ct.Structure):
    _fields_ = [("near_pairs", ct.c_longlong), ("far_work", ct.c_longlong),
                ("max_imag_residual", ct.c_double)]


class PlanInfo(ct.Structure):
    _fields_ = [
        ("d", ct.c_int), ("m_per_dim", ct.c_int), ("leaf_level", ct.c_int), ("nrhs", ct.c_int),
        ("n", ct.c_longlong), ("K", ct.c_longlong), ("boxes", ct.c_longlong * 25),
        ("near_pairs", ct.c_longlong), ("far_work", ct.c_longlong),
        ("far_work_single", ct.c_longlong), ("il_pairs", ct.c_longlong),
        ("owned_begin", ct.c_longlong), ("owned_end", ct.c_longlong),
        ("plan_seconds", ct.c_double), ("device_bytes", ct.c_longlong),
        ("stored_nodes", ct.c_longlong), ("telescoped", ct.c_int),
        ("near_sym_items", ct.c_longlong), ("near_items", ct.c_longlong),
        ("kernels", ct.c_char * 256),
    ]


class Tuning(ct.Structure):
    """blfmm_tuning (include/blfmm_gpu.h): kernel / schedule selection."""
    _fields_ = [("telescope", ct.c_int), ("graphs", ct.c_int), ("near_sym_min", ct.c_int),
                ("near_ctas_per_sm", ct.c_int), ("near_reg_cap", ct.c_int),
                ("couple_tile", ct.c_int), ("rhs_gemm", ct.c_int),
                ("half_spectrum", ct.c_int)]


# blfmm_comm_ops callbacks: (ctx, device pointer, count, [root,] stream) -> 0 / error
SUM_FN = ct.CFUNCTYPE(ct.c_int, ct.c_void_p, ct.c_void_p, ct.c_longlong, ct.c_void_p)
BCAST_FN = ct.CFUNCTYPE(ct.c_int, ct.c_void_p, ct.c_void_p, ct.c_longlong, ct.c_int, ct.c_void_p)


class CommOps(ct.Structure):
    """blfmm_comm_ops (include/blfmm_gpu.h): caller-supplied collectives."""
    _fields_ = [("ctx", ct.c_void_p), ("all_reduce_sum", SUM_FN), ("all_reduce_max", SUM_FN),
                ("broadcast", BCAST_FN)]


NCCL_ID_BYTES = 128
SOLVE_CG, SOLVE_GMRES = 1, 2


class SolveStatsC(ct.Structure):
    """blfmm_solve_stats (include/blfmm_gpu.h)."""
    _fields_ = [("method", ct.c_int), ("iterations", ct.c_int), ("matvecs", ct.c_int),
                ("converged", ct.c_int), ("residual", ct.c_double)]


class StageTimes(ct.Structure):
    _fields_ = [("ms", ct.c_double * NSTAGES), ("launches", ct.c_int * NSTAGES)]


EXPORTS = {
    # name: (restype, argtypes)
    "blfmm_last_error": (ct.c_char_p, []),
    "blfmm_last_error_value": (ct.c_double, []),
    "blfmm_abi_version": (ct.c_int, []),
    "blfmm_parse_kernel_spec": (ct.c_int, [ct.c_char_p, ct.POINTER(ct.c_int), ct.POINTER(ct.c_double)]),
    "blfmm_translation_coefficients": (ct.c_int, [ct.c_int, ct.c_int, ct.c_double, ct.c_double,
                                                  ct.c_int, ct.POINTER(ct.c_double)]),
    "blfmm_plan_create": (ct.c_int, [ct.POINTER(PlanDesc), ct.POINTER(ct.c_void_p)]),
    "blfmm_plan_destroy": (ct.c_int, [ct.c_void_p]),
    "blfmm_tuning_defaults": (None, [ct.POINTER(Tuning)]),
    "blfmm_plan_create_tuned": (ct.c_int, [ct.POINTER(PlanDesc), ct.POINTER(Tuning),
                                           ct.POINTER(ct.c_void_p)]),
    "blfmm_plan_get_info": (ct.c_int, [ct.c_void_p, ct.POINTER(PlanInfo)]),
    "blfmm_execute": (ct.c_int, [ct.c_void_p, ct.POINTER(ct.c_double), ct.POINTER(ct.c_double),
                                 ct.POINTER(Stats), ct.c_void_p]),
    "blfmm_execute_device": (ct.c_int, [ct.c_void_p, ct.c_void_p, ct.c_void_p,
                                        ct.POINTER(Stats), ct.c_void_p]),
    "blfmm_execute_single": (ct.c_int, [ct.c_void_p, ct.POINTER(ct.c_double),
                                        ct.POINTER(ct.c_double), ct.POINTER(Stats), ct.c_void_p]),
    "blfmm_get_expansions": (ct.c_int, [ct.c_void_p, ct.c_int, ct.c_int, ct.c_int,
                                        ct.POINTER(ct.c_double)]),
    "blfmm_set_keep_couple": (ct.c_int, [ct.c_void_p, ct.c_int]),
    "blfmm_set_profiling": (ct.c_int, [ct.c_void_p, ct.c_int]),
    "blfmm_get_stage_times": (ct.c_int, [ct.c_void_p, ct.POINTER(StageTimes)]),
    "blfmm_partition": (ct.c_int, [ct.POINTER(ct.c_double), ct.c_longlong, ct.c_int,
                                   ct.POINTER(ct.c_longlong)]),
    "blfmm_plan_owned_points": (ct.c_int, [ct.c_void_p, ct.POINTER(ct.c_longlong)]),
    "blfmm_plan_exchange_size": (ct.c_int, [ct.c_void_p, ct.POINTER(ct.c_longlong)]),
    "blfmm_plan_bind_exchange": (ct.c_int, [ct.c_void_p, ct.c_void_p]),
    "blfmm_execute_upsweep": (ct.c_int, [ct.c_void_p, ct.c_void_p, ct.c_void_p]),
    "blfmm_execute_downsweep": (ct.c_int, [ct.c_void_p, ct.c_void_p, ct.POINTER(Stats),
                                           ct.c_void_p]),
    "blfmm_nccl_get_unique_id": (ct.c_int, [ct.c_char_p]),
    "blfmm_solve": (ct.c_int, [ct.c_void_p, ct.c_int, ct.POINTER(ct.c_double),
                               ct.POINTER(ct.c_double), ct.c_double, ct.c_int,
                               ct.POINTER(SolveStatsC)]),
    "blfmm_solve_dense": (ct.c_int, [ct.c_int, ct.c_longlong, ct.POINTER(ct.c_double), ct.c_int,
                                     ct.c_double, ct.c_int, ct.POINTER(ct.c_double),
                                     ct.POINTER(ct.c_double), ct.c_double, ct.c_int,
                                     ct.POINTER(SolveStatsC), ct.c_int]),
    "blfmm_plan_attach_nccl": (ct.c_int, [ct.c_void_p, ct.c_char_p]),
    "blfmm_plan_attach_comm": (ct.c_int, [ct.c_void_p, ct.POINTER(CommOps)]),
    "blfmm_direct": (ct.c_int, [ct.c_int, ct.c_longlong, ct.POINTER(ct.c_double), ct.c_int,
                                ct.c_double, ct.POINTER(ct.c_double), ct.c_longlong,
                                ct.POINTER(ct.c_longlong), ct.POINTER(ct.c_double), ct.c_int]),
    "blfmm_direct_bandlimited": (ct.c_int, [ct.c_int, ct.c_longlong, ct.POINTER(ct.c_double), ct.POINTER(ct.c_double), ct.POINTER(ct.c_double), ct.c_int,
                                            ct.c_double, ct.POINTER(ct.c_double), ct.c_double, ct.c_int, ct.c_int,
                                            ct.POINTER(ct.c_double), ct.c_int]),
    "blfmm_eval_bandlimited": (ct.c_int, [ct.c_int, ct.c_int, ct.c_double, ct.c_double,
                                          ct.c_double, ct.c_int, ct.POINTER(ct.c_double)]),
    "blfmm_bandlimited_radial_table": (ct.c_int, [ct.c_int, ct.c_double, ct.c_double,
                                                  ct.c_double, ct.c_int, ct.POINTER(ct.c_double), ct.POINTER(ct.c_double)]),
}

_lib = None


def lib():
    """Load the CUDA extension (fails loudly: no CPU fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"CUDA extension {LIB_PATH} is missing; run __graft_entry__.build() "
                "(there is no CPU fallback)")
        l = ct.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            f = getattr(l, name)
            f.restype = res
            f.argtypes = args
        _lib = l
    return _lib


class BlfmmError(RuntimeError):
    pass


class InvalidArgument(BlfmmError, ValueError):
    """std::invalid_argument"""


class DomainError(BlfmmError, ArithmeticError):
    """std::domain_error"""


class LengthError(BlfmmError, ValueError):
    """std::length_error (assemble_dense's N <= 8192 cap, solver.cpp:211)"""


class AccuracyError(BlfmmError):
    """blfmm::accuracy_error (common.hpp:33-41)"""

    def __init__(self, msg, achieved):
        super().__init__(msg)
        self.achieved = achieved


class CudaError(BlfmmError):
    pass


def check(code: int):
    if code == OK:
        return
    l = lib()
    msg = l.blfmm_last_error().decode(errors="replace")
    if code == EINVAL:
        raise InvalidArgument(msg)
    if code == EDOMAIN:
        raise DomainError(msg)
    if code == EACCURACY:
        raise AccuracyError(msg, l.blfmm_last_error_value())
    if code == ENOMEM:
        raise MemoryError(msg)
    if code == ELENGTH:
        raise LengthError(msg)
    raise CudaError(f"[{code}] {msg}")
