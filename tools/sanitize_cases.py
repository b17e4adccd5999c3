"""Small solves for compute-sanitizer (memcheck / racecheck / synccheck):
heat1d two-level (TMA row loads, per-warp TMA stores, window kernel), heat1d
FAS V-cycle, Allen-Cahn (cyclic Newton Phi), 2D heat (cluster CG with DSMEM
halos, on-chip and global-scratch x), Gray-Scott (BiCGSTAB).  Tiny sizes:
every kernel family launches, nothing long-running.

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py [case ...]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_09596_b200 as T  # noqa: E402


def heat_two_level():
    app = T.Heat1D(255, manufactured_forcing=False, initial_condition=T.random_state(7, 255))
    hier = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, 257), [16], 4)
    return T.solve(app, hier, T.SolverConfig(tol=1e-10, max_iters=30, initial_guess=T.InitialGuess.Random,
                                             seed=20))


def heat_l32_fcf():
    app = T.Heat1D(4095, manufactured_forcing=False, initial_condition=T.random_state(7, 4095))
    hier = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0 / 64, 129), [16], 3)
    return T.solve(app, hier, T.SolverConfig(relaxation=T.Relaxation.FCF, tol=1e-10, max_iters=4,
                                             initial_guess=T.InitialGuess.Random, seed=20), workers=2)


def heat_fas():
    app = T.Heat1D(127, folded=True, manufactured_forcing=True)
    hier = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, 257), [4, 4], 3)
    return T.solve(app, hier, T.SolverConfig(mode=T.CycleMode.VCycle, tol=1e-10, max_iters=6,
                                             initial_guess=T.InitialGuess.Random, seed=3))


def allen_cahn():
    app = T.AllenCahn(256, 0.02, 1.0, 1e-11, 30, initial_condition=0.05 * T.random_state(3, 256))
    hier = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, 129), [4, 4], 3)
    return T.solve(app, hier, T.SolverConfig(mode=T.CycleMode.VCycle, tol=1e-9, max_iters=4,
                                             initial_guess=T.InitialGuess.Random, seed=20))


def heat2d():
    app = T.Heat2D(31, folded=False, source=T.gaussian_source(31))
    hier = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, 33), [8], 2)
    return T.solve(app, hier, T.SolverConfig(tol=1e-9, max_iters=3, initial_guess=T.InitialGuess.Random,
                                             seed=20))


def heat2d_big():
    # nx = 511: non-portable 11-CTA cluster, x / r in global scratch
    app = T.Heat2D(511, folded=True, initial_condition=T.fourier_ic(511))
    hier = T.build_hierarchy(T.TimeGrid.make(0.0, 0.001, 5), [2], 2)
    return T.solve(app, hier, T.SolverConfig(mode=T.CycleMode.VCycle, tol=1e-9, max_iters=1,
                                             initial_guess=T.InitialGuess.Random, seed=20))


def gray_scott():
    app = T.GrayScott(8)
    hier = T.build_hierarchy(T.TimeGrid.make(0.0, 2.0, 9), [4], 2)
    return T.solve(app, hier, T.SolverConfig(mode=T.CycleMode.VCycle, tol=1e-7, max_iters=2))


CASES = dict(heat_two_level=heat_two_level, heat_l32_fcf=heat_l32_fcf, heat_fas=heat_fas,
             allen_cahn=allen_cahn, heat2d=heat2d, heat2d_big=heat2d_big, gray_scott=gray_scott)

if __name__ == "__main__":
    for name in sys.argv[1:] or list(CASES):
        r = CASES[name]()
        print(name, r.report.iterations, float(r.report.residual_norms[-1]), flush=True)
