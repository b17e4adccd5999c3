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
    # the other Phi families over the same one-shard-per-process path
    elif name == "heat2d_strip":
        # strip CG, 4-CTA clusters (config 2's grid), short horizon
        app = T.Heat2D(127, folded=False, source=T.gaussian_source(127), cg_rtol=1e-12)
        hier = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0 / 64, 65), [8], 2)
        cfg = T.SolverConfig(mode=T.CycleMode.TwoLevel, tol=1e-10, max_iters=8,
                             initial_guess=T.InitialGuess.Random, seed=20)
    elif name == "heat2d_group":
        # strip CG group mode (cooperative groups exchanging through global memory)
        app = T.Heat2D(300, folded=True, source=None, cg_rtol=1e-12, initial_condition=T.fourier_ic(300))
        hier = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0 / 256, 17), [4], 2)
        cfg = T.SolverConfig(mode=T.CycleMode.VCycle, tol=1e-10, max_iters=4,
                             initial_guess=T.InitialGuess.Random, seed=20)
    elif name == "allen_cahn":
        app = T.AllenCahn(256, 0.02, 1.0, 1e-11, 30, initial_condition=0.05 * T.random_state(3, 256))
        hier = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, 129), [4, 4], 3)
        cfg = T.SolverConfig(mode=T.CycleMode.VCycle, tol=1e-9, max_iters=20,
                             initial_guess=T.InitialGuess.Random, seed=20)
    elif name == "heat1d_cluster_rows":
        # n past 5376: rows split over a 2-CTA cluster
        app = T.Heat1D(5377, folded=True, manufactured_forcing=True)
        hier = T.build_hierarchy(T.TimeGrid.make(0.0, 1e-5, 129), [4, 4], 3)
        cfg = T.SolverConfig(mode=T.CycleMode.VCycle, tol=1e-9, max_iters=20,
                             initial_guess=T.InitialGuess.Random, seed=5)
    elif name == "gray_scott":
        app = T.GrayScott(8)
        hier = T.build_hierarchy(T.TimeGrid.make(0.0, 4.0, 33), [4], 2)
        cfg = T.SolverConfig(mode=T.CycleMode.VCycle, tol=1e-7, max_iters=10)
    else:
        raise KeyError(name)
    return app, hier, cfg
