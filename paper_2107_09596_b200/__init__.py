"""B200-native AT-MGRIT hot path (arXiv 2107.09596).

The solver runs in libatmgrit.so (hand-written sm_100a CUDA kernels + a C++
host runtime behind the C ABI in include/atmgrit.h).  This package is the
reference-shaped Python binding used by tests and the benchmark.
"""
from .api import (  # noqa: F401
    AllenCahn, Application, ConfigError, ConvergenceReport, CycleDriver, CycleMode, Dahlquist,
    DivergenceError, GrayScott, Heat1D, Heat2D, Hierarchy, InitialGuess, NonlinearSolveError, NormKind,
    Relaxation, RuntimeFault, ScalarLinear, SolveResult, SolverConfig, StopReason, TempoError, TimeGrid,
    allen_cahn_ic, build_comm_groups, build_hierarchy, build_layout, fourier_ic, gaussian_source,
    make_cf_split, random_state,
    rank_ranges, run_parallel, solve, window_recvs,
)
from ._capi import LIB_PATH, lib  # noqa: F401

__all__ = [n for n in dir() if not n.startswith("_")]
