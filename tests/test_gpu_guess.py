"""Provided initial guess with atm_runtime.defer_guess: atm_setup sends only
the level-0 C rows (the default, defer_guess = 0, copies the whole guess).

Every cycle opens with an F-relaxation from the C points (kernels.cpp:7-17)
and its correction F-sweep rewrites every level-0 F row before anything reads
one, so the F values of a provided guess (solver.cpp:129-131) cannot reach
the result.  The engine therefore defers them: they are copied only if
something could read them before the first cycle (the full residual norm,
level-0 reads and writes, the kernel-level entry points, nested init).

Checks: a guess whose F rows are NaN solves BITWISE like the same guess with
finite F rows copied eagerly (the default), across cycle modes, relaxations,
families (heat, scalar, Allen-Cahn Newton, 2D heat CG, Gray-Scott BiCGSTAB)
and shard counts; every pre-cycle access sees the full guess; a cycle that
fails (Newton cap) leaves the state an eager copy would; the traffic counters
report what moved."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2107_09596_b200 as T
from helpers import device_objects

pytestmark = pytest.mark.gpu

CASES = [
    # two-level F, short trailing interval (n_points - 1 not a multiple of m)
    dict(problem="heat1d", n=255, tf=1.0, n_points=1000, m=8, k=3, folded=0, manufactured=0,
         max_iters=40, tol=1e-10),
    # two-level FCF, L = 16 rows
    dict(problem="heat1d", n=4095, tf=1.0 / 64, n_points=1025, m=16, k=8, folded=0, manufactured=0,
         relax="FCF", max_iters=30, tol=1e-10),
    # FAS V-cycle on three levels, manufactured forcing
    dict(problem="heat1d", n=127, tf=1.0, n_points=1025, m="4,4", k=3, folded=1, manufactured=1,
         mode="v-cycle", max_iters=40, tol=1e-10),
    # scalar backend
    dict(problem="dahlquist", tf=2.0, n_points=4097, m="4,4", k=2, folded=1, mode="v-cycle",
         max_iters=40, tol=1e-12),
    # Allen-Cahn: Newton warm-starts from u_prev, FAS V-cycle
    dict(problem="allen_cahn", n=256, tf=1.0, n_points=257, m="4,4", k=3, mode="v-cycle",
         max_iters=30, tol=1e-9),
    # 2D heat: CG starts from x0 = u_prev, explicit source, two-level
    dict(problem="heat2d", nx=31, tf=1.0, n_points=129, m=8, k=3, folded=0, max_iters=30, tol=1e-9),
    # Gray-Scott: Newton + BiCGSTAB
    dict(problem="gray_scott", nx=8, tf=2.0, n_points=33, m=4, k=2, mode="v-cycle", max_iters=8,
         tol=1e-7),
]


def _objects(args):
    prob = args["problem"]
    if prob in ("heat1d", "dahlquist"):
        return device_objects(dict(args, guess="provided"))
    if prob == "allen_cahn":
        app = T.AllenCahn(int(args["n"]), 0.02, 1.0, 1e-11, 30,
                          initial_condition=0.05 * T.random_state(3, int(args["n"])))
    elif prob == "heat2d":
        app = T.Heat2D(int(args["nx"]), folded=False, source=T.gaussian_source(int(args["nx"])))
    else:
        app = T.GrayScott(int(args["nx"]))
    ms = [int(x) for x in str(args["m"]).split(",")]
    hier = T.build_hierarchy(T.TimeGrid.make(0.0, float(args["tf"]), int(args["n_points"])), ms,
                             int(args["k"]))
    mode = T.CycleMode.VCycle if args.get("mode") == "v-cycle" else T.CycleMode.TwoLevel
    cfg = T.SolverConfig(mode=mode, max_iters=int(args["max_iters"]), tol=float(args["tol"]),
                         initial_guess=T.InitialGuess.Provided)
    return app, hier, cfg


def _n(args):
    p = args["problem"]
    return {"heat1d": lambda: int(args["n"]), "dahlquist": lambda: 1, "allen_cahn": lambda: int(args["n"]),
            "heat2d": lambda: int(args["nx"]) ** 2, "gray_scott": lambda: 2 * int(args["nx"]) ** 2}[p]()


def _guess(args, n, seed=0):
    npts = int(args["n_points"])
    g = np.random.default_rng(seed).uniform(-1.0, 1.0, (npts, n))
    if args["problem"] in ("allen_cahn", "gray_scott"):
        # nonlinear Phi: stay near the solution manifold (Allen-Cahn |u| < 1,
        # Gray-Scott inside the bounds check)
        g = 0.05 * g if args["problem"] == "allen_cahn" else np.clip(0.5 + 0.1 * g, 0.0, 1.0)
    return g


def _f_rows_nan(args, g):
    m = int(str(args["m"]).split(",")[0])
    h = g.copy()
    f = np.ones(len(h), bool)
    f[::m] = False
    h[f] = np.nan
    return h


def _solve(args, guess, workers, eager, monkeypatch=None):
    app, hier, cfg = _objects(args)
    cfg.provided = guess
    return T.solve(app, hier, cfg, workers=workers, defer_guess=not eager)


@pytest.mark.parametrize("args", CASES, ids=lambda a: a["problem"] + "-" + a.get("mode", "two-level"))
@pytest.mark.parametrize("workers", [1, 3])
def test_nan_f_rows_solve_bitwise_like_eager_copy(args, workers):
    n = _n(args)
    g = _guess(args, n)
    a = _solve(args, g, workers, True)
    b = _solve(args, _f_rows_nan(args, g), workers, False)
    assert a.report.iterations == b.report.iterations
    assert np.array_equal(np.array(a.report.residual_norms), np.array(b.report.residual_norms))
    assert np.array_equal(a.state, b.state)
    assert np.isfinite(b.state).all()


def _driver(args, guess, monkeypatch=None, eager=False, **kw):
    app, hier, cfg = _objects(args)
    cfg.provided = guess
    d = T.CycleDriver(app, hier, cfg, defer_guess=not eager, **kw)
    d.setup()
    return d


def test_failed_first_cycle_leaves_the_eager_state():
    # a provided guess whose first cycle raises NonlinearSolveError
    # (Allen-Cahn Newton capped at one iteration) must leave level 0 as an
    # eager copy would -- never the zero-filled F rows of a dropped deferral
    args = dict(CASES[4])
    g = _guess(args, _n(args), seed=7)
    states = []
    for eager in (True, False):
        app, hier, cfg = _objects(args)
        app = T.AllenCahn(int(args["n"]), 0.02, 1.0, 1e-14, 1,
                          initial_condition=0.05 * T.random_state(3, int(args["n"])))
        cfg.provided = g
        d = T.CycleDriver(app, hier, cfg, defer_guess=not eager)
        d.setup()
        with pytest.raises(T.NonlinearSolveError):
            d.cycle()
        states.append(d.get_level(0))
    assert np.array_equal(states[0], states[1])
    assert np.isfinite(states[1]).all() and np.any(states[1][1:] != 0.0)


def test_pre_cycle_accesses_see_the_full_guess(monkeypatch):
    args = CASES[0]
    g = _guess(args, 255, seed=3)
    # full residual norm before any cycle reads every F row
    e = _driver(args, g, monkeypatch, eager=True)
    ref_norm = e.residual_norm()
    ref_state = e.get_level(0)
    lz = _driver(args, g, monkeypatch)
    assert lz.residual_norm() == ref_norm
    # level-0 read before any cycle: the provided guess (point 0 = IC)
    lz2 = _driver(args, g, monkeypatch)
    s = lz2.get_level(0)
    assert np.array_equal(s, ref_state)
    assert np.array_equal(s[1:], g[1:])
    # kernel-level F-relaxation of one interval reads no F row, but the
    # residual of an F point does
    k1 = _driver(args, g, monkeypatch)
    k2 = _driver(args, g, monkeypatch, eager=True)
    r1 = k1.residual(0, 0, 40)
    r2 = k2.residual(0, 0, 40)
    assert np.array_equal(r1, r2)
    # a partial level-0 write before the first cycle keeps the other F rows
    w = _driver(args, g, monkeypatch)
    w.set_level(0, np.full((2, 255), 0.5), first=9)
    s = w.get_level(0)
    assert np.array_equal(s[9:11], np.full((2, 255), 0.5))
    assert np.array_equal(s[11:], g[11:])
    assert np.array_equal(s[1:9], g[1:9])


def test_nested_v_with_provided_guess(monkeypatch):
    args = dict(problem="heat1d", n=255, tf=1.0, n_points=1025, m="8,4", k=2, folded=1, manufactured=1,
                mode="nested-v", max_iters=30, tol=1e-10)
    g = _guess(args, 255, seed=4)
    a = _solve(args, g, 1, True, monkeypatch)
    b = _solve(args, g, 1, False, monkeypatch)
    assert a.report.iterations == b.report.iterations
    assert np.array_equal(a.state, b.state)


def test_host_traffic_counts_c_rows_then_readback(monkeypatch):
    args = CASES[0]
    n, npts, m = 255, 1000, 8
    g = _guess(args, n, seed=5)
    d = _driver(args, g, monkeypatch)
    h2d, d2h = d.host_traffic()
    c_rows = len(range(m, npts, m))  # C points after point 0 (the IC)
    assert (h2d, d2h) == (8 * n * c_rows, 0)
    d.iterate(2)
    assert d.host_traffic() == (8 * n * c_rows, 0)  # the cycles never needed the F rows
    d.get_level(0)
    assert d.host_traffic() == (8 * n * c_rows, 8 * n * npts)
    e = _driver(args, g, monkeypatch, eager=True)
    assert e.host_traffic() == (8 * n * (npts - 1), 0)
