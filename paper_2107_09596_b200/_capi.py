"""ctypes declaration of include/atmgrit.h and the loader of libatmgrit.so.

The product path has no fallback: if the CUDA library is missing the import
of any solver entry point raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ATM_LIB") or os.path.join(HERE, "libatmgrit.so")
MAXL = 8
ABI_VERSION = 6  # include/atmgrit.h ATM_ABI_VERSION: the structs below are its layout
_DP = C.POINTER(C.c_double)
_IP = C.POINTER(C.c_int)


class atm_problem(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("n", C.c_int), ("folded", C.c_int),
        ("x0", C.c_double), ("x1", C.c_double), ("manufactured", C.c_int),
        ("lam", C.c_double), ("u0", C.c_double),
        ("n_mult", C.c_int), ("mult", C.c_double * MAXL),
        ("fine_forcing", _DP), ("n_ff", C.c_int),
        ("eps", C.c_double), ("length", C.c_double),
        ("newton_tol", C.c_double), ("newton_max", C.c_int),
        ("nx", C.c_int), ("cg_rtol", C.c_double), ("cg_max", C.c_int),
        ("source", _DP), ("ic", _DP),
        ("gs_domain", C.c_double), ("gs_feed", C.c_double), ("gs_kill", C.c_double),
        ("gs_du", C.c_double), ("gs_dv", C.c_double), ("gs_linear_tol", C.c_double),
        ("gs_reaction", C.c_int), ("gs_bounds_check", C.c_int),
        ("gs_bound_lo", C.c_double), ("gs_bound_hi", C.c_double),
    ]


class atm_grid(C.Structure):
    _fields_ = [("t0", C.c_double), ("tf", C.c_double), ("n_points", C.c_int),
                ("n_m", C.c_int), ("m", C.c_int * MAXL), ("k", C.c_int)]


class atm_solver(C.Structure):
    _fields_ = [("mode", C.c_int), ("relaxation", C.c_int), ("nu", C.c_int),
                ("max_iters", C.c_int), ("tol", C.c_double), ("norm", C.c_int),
                ("functional_w", _DP), ("initial_guess", C.c_int), ("seed", C.c_uint64),
                ("constant_value", _DP), ("provided", _DP), ("coarse_substeps", C.c_int),
                ("functional_kind", C.c_int)]


class atm_runtime(C.Structure):
    _fields_ = [("device", C.c_int), ("n_shards", C.c_int), ("world_size", C.c_int),
                ("rank", C.c_int), ("nccl_id", C.c_void_p), ("storage", C.c_int),
                ("trace", C.c_int), ("reuse_relax", C.c_int), ("defer_guess", C.c_int),
                ("timeout_ms", C.c_int)]


class atm_report(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("stop_reason", C.c_int),
                ("total_seconds", C.c_double), ("dof_steps", C.c_double),
                ("setup_seconds", C.c_double)]


# exported symbol -> (restype, argtypes); the authoritative list is atmgrit.h
SIGNATURES = {
    "atm_abi_version": (C.c_int, []),
    "atm_create_error": (C.c_char_p, []),
    "atm_device_count": (C.c_int, []),
    "atm_create": (C.c_int, [C.POINTER(atm_problem), C.POINTER(atm_grid), C.POINTER(atm_solver),
                             C.POINTER(atm_runtime), C.POINTER(C.c_void_p)]),
    "atm_destroy": (None, [C.c_void_p]),
    "atm_last_error": (C.c_char_p, [C.c_void_p]),
    "atm_setup": (C.c_int, [C.c_void_p]),
    "atm_nested_init": (C.c_int, [C.c_void_p]),
    "atm_cycle": (C.c_int, [C.c_void_p]),
    "atm_residual_norm": (C.c_int, [C.c_void_p, _DP]),
    "atm_solve": (C.c_int, [C.c_void_p, C.POINTER(atm_report), _DP, _DP]),
    "atm_iterate": (C.c_int, [C.c_void_p, C.c_int, _DP]),
    "atm_get_level": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, _DP]),
    "atm_set_level": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, _DP]),
    "atm_level_points": (C.c_int, [C.c_void_p, C.c_int]),
    "atm_vector_size": (C.c_int, [C.c_void_p]),
    "atm_n_levels": (C.c_int, [C.c_void_p]),
    "atm_apply_phi": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, _DP, _DP]),
    "atm_forcing": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, _DP]),
    "atm_kernel_f_relax": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int]),
    "atm_kernel_c_relax": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int]),
    "atm_kernel_residual": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, _DP]),
    "atm_phase_times": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int, _DP, C.c_int]),
    "atm_last_iteration_stats": (C.c_int, [C.c_void_p, _IP, _DP]),
    "atm_inner_iterations": (C.c_int, [C.c_void_p, C.POINTER(C.c_ulonglong)]),
    "atm_host_traffic": (C.c_int, [C.c_void_p, C.POINTER(C.c_ulonglong), C.POINTER(C.c_ulonglong)]),
    "atm_phase_counts": (C.c_int, [C.c_void_p, _IP, C.c_int]),
    "atm_iterate_timed": (C.c_int, [C.c_void_p, C.c_int, _DP, _DP]),
    "atm_host_register": (C.c_int, [C.c_void_p, C.c_size_t]),
    "atm_host_unregister": (C.c_int, [C.c_void_p]),
    "atm_random_state": (None, [C.c_uint64, C.c_int, _DP]),
    "atm_build_layout": (C.c_int, [C.POINTER(atm_grid), C.c_int, _IP, _IP, _IP, _IP]),
    "atm_rank_ranges": (C.c_int, [C.POINTER(atm_grid), C.c_int, C.c_int] + [_IP] * 8),
    "atm_window_recvs": (C.c_int, [C.POINTER(atm_grid), C.c_int, C.c_int, _IP, C.c_int]),
    "atm_nccl_unique_id": (C.c_int, [C.c_void_p]),
}

_lib = None


class LibraryMissing(RuntimeError):
    pass


def lib():
    """Load libatmgrit.so; raise loudly when it is absent (no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise LibraryMissing(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                " (the AT-MGRIT path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        if L.atm_abi_version() != ABI_VERSION:
            raise LibraryMissing(f"{LIB_PATH} has ABI {L.atm_abi_version()}, these bindings expect "
                                 f"{ABI_VERSION}: rebuild it")
        _lib = L
    return _lib


def ptr(a):
    return a.ctypes.data_as(_DP)
