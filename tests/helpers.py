"""Translate one case description (the key=value args of the compiled
reference driver, oracle/ref_driver.cpp) into (a) device-side objects of
paper_2107_09596_b200 and (b) the C oracle restatement's dicts."""
from __future__ import annotations

import numpy as np

import paper_2107_09596_b200 as T
from oracle import oracle as O


def _ms(args):
    m = args.get("m", 4)
    return [int(x) for x in str(m).split(",")]


def _functional(args, files):
    """SolverConfig.functional of a tempo_ref case (ref_driver.cpp functional=)."""
    fk = args.get("functional", "first")
    if fk == "norm2":
        return "norm2"
    if fk == "weights":
        return files["w_file"]
    w = np.zeros(int(args.get("n", 1)) if args.get("problem", "heat1d") == "heat1d" else 1)
    w[0] = 1.0  # u[0]
    return w


def device_objects(args, ic=None, ff=None, files=None):
    prob = args.get("problem", "heat1d")
    if prob == "heat1d":
        app = T.Heat1D(int(args.get("n", 1025)), float(args.get("x0", 0.0)), float(args.get("x1", 1.0)),
                       folded=bool(int(args.get("folded", 0))),
                       manufactured_forcing=bool(int(args.get("manufactured", 1))),
                       initial_condition=ic)
    elif prob == "dahlquist":
        app = T.Dahlquist(float(args.get("lambda", -1.0)), float(args.get("u0", 1.0)),
                          folded=bool(int(args.get("folded", 0))))
    else:
        mult = [float(x) for x in str(args.get("mult", "0.5,0.25")).split(",")]
        app = T.ScalarLinear(mult, float(args.get("u0", 1.0)), bool(int(args.get("folded", 0))), ff)
    hier = T.build_hierarchy(T.TimeGrid.make(float(args.get("t0", 0.0)), float(args.get("tf", 1.0)),
                                             int(args.get("n_points", 33))), _ms(args), int(args.get("k", 2)))
    mode = {"two-level": T.CycleMode.TwoLevel, "v-cycle": T.CycleMode.VCycle,
            "nested-v": T.CycleMode.NestedV}[args.get("mode", "two-level")]
    guess = {"constant": T.InitialGuess.Constant, "random": T.InitialGuess.Random,
             "provided": T.InitialGuess.Provided}[args.get("guess", "constant")]
    cfg = T.SolverConfig(mode=mode, relaxation=T.Relaxation.FCF if args.get("relax", "F") == "FCF" else T.Relaxation.F,
                         nu=int(args.get("nu", 1)), max_iters=int(args.get("max_iters", 100)),
                         tol=float(args.get("tol", 1e-7)), initial_guess=guess, seed=int(args.get("seed", 0)),
                         coarse_substeps=int(args.get("substeps", 1)))
    if args.get("norm") == "functional":
        cfg.norm = T.NormKind.FunctionalChange
        cfg.functional = _functional(args, files or {})
    return app, hier, cfg


def oracle_driver(args, ic=None, ff=None, **over):
    prob = args.get("problem", "heat1d")
    if prob == "heat1d":
        p = dict(kind=O.HEAT1D, n=int(args.get("n", 1025)), x0=float(args.get("x0", 0.0)),
                 x1=float(args.get("x1", 1.0)), folded=int(args.get("folded", 0)),
                 manufactured=int(args.get("manufactured", 1)), ic=ic)
    elif prob == "dahlquist":
        p = dict(kind=O.DAHLQUIST, lam=float(args.get("lambda", -1.0)), u0=float(args.get("u0", 1.0)),
                 folded=int(args.get("folded", 0)))
    else:
        p = dict(kind=O.SCALAR, mult=[float(x) for x in str(args.get("mult", "0.5,0.25")).split(",")],
                 u0=float(args.get("u0", 1.0)), folded=int(args.get("folded", 0)), fine_forcing=ff)
    g = dict(t0=float(args.get("t0", 0.0)), tf=float(args.get("tf", 1.0)),
             n_points=int(args.get("n_points", 33)), m=_ms(args), k=int(args.get("k", 2)))
    mode = {"two-level": O.TWO_LEVEL, "v-cycle": O.VCYCLE, "nested-v": O.NESTED_V}[args.get("mode", "two-level")]
    guess = {"constant": O.GUESS_CONSTANT, "random": O.GUESS_RANDOM,
             "provided": O.GUESS_PROVIDED}[args.get("guess", "constant")]
    s = dict(mode=mode, relaxation=O.RELAX_FCF if args.get("relax", "F") == "FCF" else O.RELAX_F,
             nu=int(args.get("nu", 1)), max_iters=int(args.get("max_iters", 100)),
             tol=float(args.get("tol", 1e-7)), initial_guess=guess, seed=int(args.get("seed", 0)),
             coarse_substeps=int(args.get("substeps", 1)))
    s.update(over)
    return O.Driver(p, g, s)


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
