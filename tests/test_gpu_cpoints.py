"""C-point-only level-0 storage (atm_runtime.storage = ATM_STORE_CPOINTS;
SURVEY 7.2 item 1: config 4's full fine grid does not fit one GPU).  Level 0
keeps only its C points; its F values are, by definition, the F-relaxation of
their interval's C point and are recomputed on read.  With F-relaxation every
cycle ends with exactly that F-sweep, so histories, iteration counts and the
assembled state must be BITWISE those of full storage (the same kernels do the
same arithmetic; only dead F-row stores disappear)."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2107_09596_b200 as T
from helpers import device_objects

pytestmark = pytest.mark.gpu


def _same(a, b):
    assert a.report.iterations == b.report.iterations
    assert np.array_equal(np.array(a.report.residual_norms), np.array(b.report.residual_norms))
    assert np.array_equal(a.state, b.state)


HEAT_CASES = [
    # two-level (explicit, unforced: no stored level-0 forcing), several chunk
    # lengths (L = 16 / 32 rows)
    dict(problem="heat1d", n=1025, tf=1.0, n_points=2049, m=16, k=4, folded=0, manufactured=0,
         guess="random", seed=21, max_iters=60, tol=1e-10),
    dict(problem="heat1d", n=4095, tf=1.0 / 64, n_points=1025, m=16, k=8, folded=0, manufactured=0,
         guess="random", seed=5, max_iters=60, tol=1e-10),
    # short trailing interval, constant guess
    dict(problem="heat1d", n=63, tf=1.0, n_points=1000, m=8, k=3, folded=0, manufactured=0,
         guess="constant", max_iters=60, tol=1e-10),
    # FAS V-cycle and nested-V on three levels
    dict(problem="heat1d", n=255, tf=1.0, n_points=1025, m="4,4", k=3, folded=1, manufactured=1,
         mode="v-cycle", guess="random", seed=7, max_iters=60, tol=1e-10),
    dict(problem="heat1d", n=255, tf=1.0, n_points=1025, m="8,4", k=2, folded=1, manufactured=1,
         mode="nested-v", guess="random", seed=8, max_iters=60, tol=1e-10),
    # scalar families (row kernels of the scalar backend)
    dict(problem="dahlquist", tf=2.0, n_points=4097, m="4,4", k=2, folded=1, mode="v-cycle",
         guess="random", seed=3, max_iters=60, tol=1e-12),
    dict(problem="scalar", mult="0.9,0.6", u0=1.0, folded=0, n_points=513, m=8, k=3,
         guess="random", seed=2, max_iters=60, tol=1e-13),
]


@pytest.mark.parametrize("args", HEAT_CASES)
@pytest.mark.parametrize("workers", [1, 3])
def test_cpoint_storage_bitwise_equals_full_storage(args, workers):
    app, hier, cfg = device_objects(args)
    a = T.solve(app, hier, cfg, workers=workers)
    b = T.solve(app, hier, cfg, workers=workers, cpoint_storage=True)
    _same(a, b)


def test_cpoint_storage_with_relax_reuse():
    args = dict(problem="heat1d", n=1025, tf=1.0, n_points=4097, m=16, k=4, folded=0, manufactured=0,
                guess="random", seed=11, max_iters=60, tol=1e-11)
    app, hier, cfg = device_objects(args)
    a = T.solve(app, hier, cfg)
    b = T.solve(app, hier, cfg, cpoint_storage=True, reuse_relax=True)
    _same(a, b)


FAS_REUSE_CASES = [
    # FAS V-cycles: the level-0 opening F-sweep repeats the previous cycle's
    # level-0 correction sweep (the coarser levels are re-injected each cycle)
    dict(problem="heat1d", n=255, tf=1.0, n_points=1025, m="4,4", k=3, folded=1, manufactured=1,
         mode="v-cycle", guess="random", seed=7, max_iters=60, tol=1e-10),
    dict(problem="heat1d", n=1025, tf=1.0, n_points=2049, m="16", k=4, folded=1, manufactured=1,
         mode="v-cycle", guess="random", seed=9, max_iters=60, tol=1e-10),
    dict(problem="heat1d", n=255, tf=1.0, n_points=1025, m="8,4", k=2, folded=1, manufactured=1,
         mode="nested-v", guess="random", seed=8, max_iters=60, tol=1e-10),
    dict(problem="heat1d", n=127, tf=1.0, n_points=1025, m="4,4,4", k=2, folded=1, manufactured=0,
         mode="v-cycle", guess="random", seed=5, substeps=2, max_iters=60, tol=1e-10),
    dict(problem="dahlquist", tf=2.0, n_points=4097, m="4,4", k=2, folded=1, mode="v-cycle",
         guess="random", seed=3, max_iters=60, tol=1e-12),
]


@pytest.mark.parametrize("args", FAS_REUSE_CASES)
@pytest.mark.parametrize("workers", [1, 3])
def test_relax_reuse_in_fas_vcycles_bitwise_equals_full_cycles(args, workers):
    app, hier, cfg = device_objects(args)
    a = T.solve(app, hier, cfg, workers=workers)
    b = T.solve(app, hier, cfg, workers=workers, reuse_relax=True)
    _same(a, b)
    if a.report.iterations > 1:
        assert b.report.dof_steps < a.report.dof_steps
    if not int(args.get("manufactured", 0)) or int(args.get("folded", 0)):
        _same(a, T.solve(app, hier, cfg, workers=workers, reuse_relax=True, cpoint_storage=True))


def test_relax_reuse_fas_allen_cahn_heat2d_gray_scott():
    ic = 0.05 * T.random_state(3, 256)
    app = T.AllenCahn(256, 0.02, 1.0, 1e-12, 30, initial_condition=ic)
    hier = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, 513), [8, 4], 3)
    cfg = T.SolverConfig(mode=T.CycleMode.VCycle, max_iters=40, tol=1e-9,
                         initial_guess=T.InitialGuess.Random, seed=20)
    a = T.solve(app, hier, cfg, workers=2)
    _same(a, T.solve(app, hier, cfg, workers=2, reuse_relax=True))
    _same(a, T.solve(app, hier, cfg, workers=2, reuse_relax=True, cpoint_storage=True))
    app = T.Heat2D(31, folded=True, source=T.gaussian_source(31), cg_rtol=1e-12, cg_max=10000)
    hier = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, 257), [8, 4], 2)
    for mode in (T.CycleMode.VCycle, T.CycleMode.NestedV):
        cfg = T.SolverConfig(mode=mode, max_iters=40, tol=1e-9, initial_guess=T.InitialGuess.Random, seed=20)
        a = T.solve(app, hier, cfg)
        _same(a, T.solve(app, hier, cfg, reuse_relax=True))
        _same(a, T.solve(app, hier, cfg, reuse_relax=True, cpoint_storage=True))
    app = T.GrayScott(16)
    hier = T.build_hierarchy(T.TimeGrid.make(0.0, 8.0, 129), [8], 4)
    cfg = T.SolverConfig(mode=T.CycleMode.NestedV, max_iters=30, tol=1e-7)
    _same(T.solve(app, hier, cfg), T.solve(app, hier, cfg, reuse_relax=True))


def test_relax_reuse_fas_invalidated_by_set_level():
    args = dict(problem="heat1d", n=63, tf=1.0, n_points=257, m="4,4", k=3, folded=1, manufactured=1,
                mode="v-cycle", guess="random", seed=4, max_iters=20, tol=1e-14)
    app, hier, cfg = device_objects(args)
    drv_a = T.CycleDriver(app, hier, cfg)
    drv_b = T.CycleDriver(app, hier, cfg, reuse_relax=True)
    for d in (drv_a, drv_b):
        d.setup()
        d.iterate(2)
        u = d.get_level(0)
        u[5:40] *= 0.5  # perturb F and C points between cycles
        d.set_level(0, u)
    assert np.array_equal(drv_a.iterate(3), drv_b.iterate(3))
    assert np.array_equal(drv_a.get_level(0), drv_b.get_level(0))


def test_cpoint_storage_provided_guess_and_partial_reads():
    args = dict(problem="heat1d", n=127, tf=1.0, n_points=801, m=8, k=3, folded=0, manufactured=0,
                guess="provided", max_iters=4, tol=1e-300)
    app, hier, cfg = device_objects(args)
    rng = np.random.default_rng(0)
    cfg.provided = rng.standard_normal((801, 127))
    da = T.CycleDriver(app, hier, cfg)
    db = T.CycleDriver(app, hier, cfg, cpoint_storage=True)
    for d in (da, db):
        d.setup()
    # before any cycle the held C points (after point 0, the initial
    # condition) are the provided ones
    cp = db.get_level(0)[8::8]
    assert np.array_equal(cp, cfg.provided[8::8])
    assert np.array_equal(da.iterate(4), db.iterate(4))
    for first, count in [(0, 801), (3, 5), (17, 100), (792, 9), (800, 1)]:
        assert np.array_equal(da.get_level(0, first=first, count=count),
                              db.get_level(0, first=first, count=count)), (first, count)
    # the full residual norm: F residuals are zero by construction in both
    assert da.residual_norm() == db.residual_norm()


def test_cpoint_storage_chunked_readback():
    # level-0 reads rebuild F rows through a bounded scratch block (~1 GiB):
    # n = 4095 rows of 32 KiB, m = 16 -> 2048 intervals per chunk, 4 chunks
    args = dict(problem="heat1d", n=4095, tf=1.0 / 64, n_points=8 * 2048 + 1, m=16, k=8, folded=0,
                manufactured=0, guess="random", seed=9, max_iters=3, tol=1e-300)
    app, hier, cfg = device_objects(args)
    a = T.solve(app, hier, cfg)
    b = T.solve(app, hier, cfg, cpoint_storage=True)
    _same(a, b)


def test_cpoint_storage_allen_cahn_and_heat2d():
    ic = 0.05 * T.random_state(3, 256)
    app = T.AllenCahn(256, 0.02, 1.0, 1e-12, 30, initial_condition=ic)
    hier = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, 513), [8, 4], 3)
    cfg = T.SolverConfig(mode=T.CycleMode.VCycle, max_iters=40, tol=1e-9,
                         initial_guess=T.InitialGuess.Random, seed=20)
    _same(T.solve(app, hier, cfg, workers=2), T.solve(app, hier, cfg, workers=2, cpoint_storage=True))
    app = T.Heat2D(31, folded=True, source=T.gaussian_source(31), cg_rtol=1e-12, cg_max=10000)
    hier = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, 257), [8, 4], 2)
    cfg = T.SolverConfig(mode=T.CycleMode.NestedV, max_iters=40, tol=1e-9,
                         initial_guess=T.InitialGuess.Random, seed=20)
    _same(T.solve(app, hier, cfg), T.solve(app, hier, cfg, cpoint_storage=True))


def test_cpoint_storage_gray_scott():
    app = T.GrayScott(16)
    hier = T.build_hierarchy(T.TimeGrid.make(0.0, 8.0, 129), [8], 4)
    cfg = T.SolverConfig(mode=T.CycleMode.NestedV, max_iters=30, tol=1e-7)
    _same(T.solve(app, hier, cfg), T.solve(app, hier, cfg, cpoint_storage=True))


def test_cpoint_storage_set_level_writes_c_points():
    args = dict(problem="heat1d", n=63, tf=1.0, n_points=257, m=8, k=3, folded=0, manufactured=0,
                guess="random", seed=4, max_iters=20, tol=1e-14)
    app, hier, cfg = device_objects(args)
    da = T.CycleDriver(app, hier, cfg)
    db = T.CycleDriver(app, hier, cfg, cpoint_storage=True)
    for d in (da, db):
        d.setup()
        d.iterate(2)
        u = d.get_level(0)
        u[::8] *= 0.5  # perturb C points between cycles (F values follow from them)
        d.set_level(0, u)
    assert np.array_equal(da.iterate(3), db.iterate(3))
    assert np.array_equal(da.get_level(0), db.get_level(0))


@pytest.mark.parametrize("bad", ["fcf", "stored_forcing", "kernel_entry"])
def test_cpoint_storage_config_errors(bad):
    args = dict(problem="heat1d", n=63, tf=1.0, n_points=257, m=8, k=3, folded=0, manufactured=0,
                guess="random", seed=4, max_iters=5, tol=1e-14)
    if bad == "fcf":
        args["relax"] = "FCF"
    if bad == "stored_forcing":
        args["manufactured"] = 1  # explicit forcing is stored per level-0 point
    app, hier, cfg = device_objects(args)
    if bad == "kernel_entry":
        d = T.CycleDriver(app, hier, cfg, cpoint_storage=True)
        with pytest.raises(T.ConfigError):
            d.f_relax(0, 0, 2)
        return
    with pytest.raises(T.ConfigError):
        T.CycleDriver(app, hier, cfg, cpoint_storage=True)
