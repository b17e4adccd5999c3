"""Problem cases shared by the multi-process GPU test and its workers."""
import numpy as np

import paper_2107_09596_b200 as T


def build_case(name):
    if name == "two_level":
        app = T.Heat1D(63, manufactured_forcing=True)
        hier = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, 1025), [16], 4)
        cfg = T.SolverConfig(mode=T.CycleMode.TwoLevel, tol=1e-9, max_iters=60,
                             initial_guess=T.InitialGuess.Random, seed=5)
    elif name == "fas_vcycle":
        app = T.Heat1D(47, folded=True, manufactured_forcing=True)
        hier = T.build_hierarchy(T.TimeGrid.make(0.0, 2.0, 257), [4, 4], 3)
        cfg = T.SolverConfig(mode=T.CycleMode.VCycle, tol=1e-9, max_iters=40,
                             initial_guess=T.InitialGuess.Random, seed=5, coarse_substeps=2)
    elif name == "nested_fcf":
        app = T.Heat1D(33, folded=True, manufactured_forcing=True)
        hier = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, 257), [4, 4], 4)
        cfg = T.SolverConfig(mode=T.CycleMode.NestedV, relaxation=T.Relaxation.FCF, tol=1e-9,
                             max_iters=40, initial_guess=T.InitialGuess.Random, seed=3)
    elif name == "global_coarse":
        # k >= N_T + 1: the nested init runs the sequential cross-shard chain
        app = T.Heat1D(33, folded=True, manufactured_forcing=True)
        hier = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, 129), [8], 40)
        cfg = T.SolverConfig(mode=T.CycleMode.NestedV, tol=1e-9, max_iters=40,
                             initial_guess=T.InitialGuess.Random, seed=3)
    else:
        raise KeyError(name)
    return app, hier, cfg
