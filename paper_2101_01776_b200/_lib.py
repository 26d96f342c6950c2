"""ctypes binding of the C ABI in include/irkg.h (libirkg.so, built in-tree).

There is no CPU fallback: if the shared library is missing or no CUDA
device is usable, every entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IRKG_LIB") or os.path.join(HERE, "libirkg.so")

MAX_STAGES = 8
MAX_NEWTON = 512
MAX_BLOCK_RECORDS = 4096

OK = 0
ERR_VALUE = -1
ERR_CONFIG = -2
ERR_STAGE_SOLVE = -3
ERR_STEP_FAILURE = -4
ERR_BREAKDOWN = -5
ERR_CUDA = -6
ERR_INDEX = -7
ERR_SINGULAR = -8
INNER_EXACT = 0
INNER_MG = -1


class Problem(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("nx", C.c_int),
        ("ny", C.c_int),
        ("nz", C.c_int),
        ("length", C.c_double),
        ("nu", C.c_double),
        ("c", C.c_double),
        ("lam", C.c_double),
        ("mu", C.c_double),
        ("length_y", C.c_double),
        ("length_z", C.c_double),
    ]


S = MAX_STAGES


class Tableau(C.Structure):
    _fields_ = [
        ("s", C.c_int),
        ("a0", C.c_double * (S * S)),
        ("b0", C.c_double * S),
        ("c0", C.c_double * S),
        ("q", C.c_double * (S * S)),
        ("r", C.c_double * (S * S)),
        ("d", C.c_double * (S * S * S)),
        ("nblocks", C.c_int),
        ("blk_offset", C.c_int * S),
        ("blk_size", C.c_int * S),
        ("blk_eta", C.c_double * S),
        ("blk_beta", C.c_double * S),
        ("blk_phi", C.c_double * S),
    ]


class Solver(C.Structure):
    _fields_ = [
        ("variant", C.c_int),
        ("newton_rtol", C.c_double),
        ("newton_maxit", C.c_int),
        ("newton_abs_floor", C.c_double),
        ("krylov_rtol", C.c_double),
        ("krylov_maxit", C.c_int),
        ("restart", C.c_int),
        ("gamma_mode", C.c_int),
        ("gamma_custom", C.c_double),
        ("inner", C.c_int),
        ("jacobian_refresh", C.c_int),
        ("variant0_stage", C.c_int),
    ]


class KrylovReportC(C.Structure):
    _fields_ = [
        ("iterations", C.c_int),
        ("converged", C.c_int),
        ("precond_applications", C.c_int),
        ("n_residuals", C.c_int),
        ("residual_capacity", C.c_int),
        ("residuals", C.POINTER(C.c_double)),
    ]


class StepStatsC(C.Structure):
    _fields_ = [
        ("newton_iterations", C.c_int),
        ("krylov_iterations", C.c_int),
        ("precond_applications", C.c_int),
        ("jacobian_assemblies", C.c_int),
        ("converged", C.c_int),
        ("n_residuals", C.c_int),
        ("residual_history", C.c_double * (MAX_NEWTON + 1)),
        ("n_block_records", C.c_int),
        ("block_offset", C.c_int * MAX_BLOCK_RECORDS),
        ("block_iterations", C.c_int * MAX_BLOCK_RECORDS),
        ("wall_time", C.c_double),
        ("fail_block_offset", C.c_int),
        ("fail_report", KrylovReportC),
        ("differential_solves", C.c_int),
        ("constraint_solves", C.c_int),
        ("constraint_residual", C.c_double),
    ]


class Counters(C.Structure):
    _fields_ = [
        ("kernel_launches", C.c_int64),
        ("arnoldi_iterations", C.c_int64),
        ("cgs_bytes", C.c_double),
        ("cgs_time_ms", C.c_double),
        ("cgs_launches", C.c_int64),
        ("precond_bytes", C.c_double),
        ("op_bytes", C.c_double),
        ("precond_time_ms", C.c_double),
        ("op_time_ms", C.c_double),
        ("halo_exchanges", C.c_int64),
        ("arnoldi_ms_1x1", C.c_double),
        ("arnoldi_ms_2x2", C.c_double),
        ("cycle_end_ms", C.c_double),
        ("newton_gap_ms", C.c_double),
        ("block_gap_ms", C.c_double),
    ]


ALLREDUCE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_int)
HALO_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                      C.c_longlong)
ALLTOALL_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p, C.c_longlong)


class OpField(C.Structure):
    _fields_ = [("a_dev", C.c_void_p), ("sigma", C.c_double)]


_P = C.c_void_p
_D = C.c_double
_I = C.c_int

_SIGS = {
    "irkg_last_error": (C.c_char_p, []),
    "irkg_version": (C.c_char_p, []),
    "irkg_create": (_I, [C.POINTER(_P), C.POINTER(Problem), _I, _P, _P, _I, _I]),
    "irkg_create_callback": (
        _I, [C.POINTER(_P), C.POINTER(Problem), _I, _P, _I, _I, ALLREDUCE_FN, HALO_FN, _P]
    ),
    "irkg_set_alltoall_callback": (_I, [_P, ALLTOALL_FN]),
    "irkg_destroy": (_I, [_P]),
    "irkg_get_local_extent": (_I, [_P, C.POINTER(_I), C.POINTER(_I), C.POINTER(_I)]),
    "irkg_nccl_unique_id": (_I, [_P]),
    "irkg_set_tableau": (_I, [_P, C.POINTER(Tableau)]),
    "irkg_set_solver": (_I, [_P, C.POINTER(Solver)]),
    "irkg_set_timing": (_I, [_P, _I]),
    "irkg_get_counters": (_I, [_P, C.POINTER(Counters)]),
    "irkg_probe_phase": (_I, [_P, _I, _I, _I, C.POINTER(C.c_double)]),
    "irkg_dirk_step": (_I, [_P, _P, C.c_double, C.c_double, C.POINTER(StepStatsC)]),
    "irkg_stage_residual": (_I, [_P, _P, _P, _D, _D, _P, C.POINTER(_D)]),
    "irkg_newton_step": (_I, [_P, _P, _P, _D, _D, C.POINTER(StepStatsC)]),
    "irkg_step": (_I, [_P, _P, _D, _D, C.POINTER(StepStatsC)]),
    "irkg_step_host": (_I, [_P, _P, _D, _D, C.POINTER(StepStatsC)]),
    "irkg_step_host_out": (_I, [_P, _P, _P, _D, _D, C.POINTER(StepStatsC)]),
    "irkg_linearize": (_I, [_P, _P, _I, _P, _P, C.POINTER(_D)]),
    "irkg_block2x2_apply": (
        _I,
        [_P, _D, _D, _D, _D, C.POINTER(OpField), C.POINTER(OpField), C.POINTER(OpField),
         C.POINTER(OpField), _P, _P],
    ),
    "irkg_block2x2_precond": (
        _I, [_P, _D, _D, _D, _D, _D, _I, C.POINTER(OpField), C.POINTER(OpField), _P, _P]
    ),
    "irkg_shifted_solve": (_I, [_P, _D, _D, _I, C.POINTER(OpField), _P, _P]),
    "irkg_block_gmres": (
        _I,
        [_P, _I, _D, _D, _D, _D, _D, _I, C.POINTER(OpField), C.POINTER(OpField),
         C.POINTER(OpField), C.POINTER(OpField), _P, _P, _D, _I, _I, C.POINTER(KrylovReportC)],
    ),
    "irkg_prepare_linearization": (_I, [_P, _P, _P, _D]),
    "irkg_transformed_solve": (_I, [_P, _D, _P, _P, C.POINTER(StepStatsC)]),
    "irkg_set_variant_jacobian": (_I, [_P, C.POINTER(OpField), _I, C.POINTER(C.c_int),
                                       C.POINTER(C.c_int), C.POINTER(OpField)]),
    "irkg_operator_apply": (_I, [_P, C.POINTER(OpField), _P, _P]),
    "irkg_rhs": (_I, [_P, _P, _D, _P]),
    "irkg_rc_gmres_begin": (_I, [_P, C.c_longlong, _P, _P, _P, _P, _P, _D, _I, _I, _I]),
    "irkg_rc_gmres_next": (_I, [_P, C.POINTER(C.c_int)]),
    "irkg_rc_gmres_report": (_I, [_P, C.POINTER(KrylovReportC)]),
    "irkg_dae_stage_residual": (_I, [_P, _P, _P, _D, _D, _P, C.POINTER(_D)]),
    "irkg_dae_step": (_I, [_P, _P, _D, _D, C.POINTER(StepStatsC)]),
    "irkg_dae_step_host": (_I, [_P, _P, _D, _D, C.POINTER(StepStatsC)]),
    "irkg_dae_constraint_norm": (_I, [_P, _P, C.POINTER(_D)]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load():
    """Load libirkg.so (raises loudly; there is no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"CUDA engine {LIB_PATH} is missing: run `python -m paper_2101_01776_b200._build` "
            "(there is no CPU fallback)"
        )
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error():
    return load().irkg_last_error().decode(errors="replace")
