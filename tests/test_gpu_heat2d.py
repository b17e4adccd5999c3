"""2D heat (BASELINE configs 2 and 4) on the device vs the C oracle.

No reference Phi exists for this family: oracle/atm_oracle.c
h2_solve restates backward Euler with the 5-point Laplacian and plain CG
(|r| <= rtol |b| from x0 = u_prev).  The device runs the same CG per
thread-block cluster (heat2d_cg.cu) with fixed-order, rank-ordered
reductions, so only the summation order of the dot products differs; the
bar is the solver's: same MGRIT iteration count, final u within 1e-10
relative l2.
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_2107_09596_b200 as T
from helpers import rel_l2
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _pair(nx, n_points, tf, ms, k, mode="two-level", folded=False, source=True, ic="zero",
          tol=1e-9, max_iters=60, cg_max=10000, substeps=1, relax="F"):
    n = nx * nx
    f = T.gaussian_source(nx) if source else None
    u0 = T.fourier_ic(nx) if ic == "fourier" else None
    app = T.Heat2D(nx, folded=folded, source=f, cg_rtol=1e-12, cg_max=cg_max, initial_condition=u0)
    hier = T.build_hierarchy(T.TimeGrid.make(0.0, tf, n_points), ms, k)
    cm = {"two-level": T.CycleMode.TwoLevel, "v-cycle": T.CycleMode.VCycle,
          "nested-v": T.CycleMode.NestedV}[mode]
    cfg = T.SolverConfig(mode=cm, relaxation=T.Relaxation.FCF if relax == "FCF" else T.Relaxation.F,
                         max_iters=max_iters, tol=tol, initial_guess=T.InitialGuess.Random, seed=20,
                         coarse_substeps=substeps)
    om = {"two-level": O.TWO_LEVEL, "v-cycle": O.VCYCLE, "nested-v": O.NESTED_V}[mode]
    orc = O.Driver(dict(kind=O.HEAT2D, n=n, nx=nx, folded=int(folded), source=f, ic=u0,
                        cg_rtol=1e-12, cg_max=cg_max),
                   dict(tf=tf, n_points=n_points, m=list(ms), k=k),
                   dict(mode=om, relaxation=O.RELAX_FCF if relax == "FCF" else O.RELAX_F,
                        max_iters=max_iters, tol=tol, initial_guess=O.GUESS_RANDOM, seed=20,
                        coarse_substeps=substeps))
    return app, hier, cfg, orc


# strip CG (heat2d_cg.cu): nx = 1, 7, 31, 63 one CTA; 127 a 4-CTA cluster
# (config 2's grid); 200, 255 clusters of 13 and 16 CTAs; 300 and 511 group
# mode (cooperative groups of 22 and 37 CTAs exchanging through global
# memory; 511 is config 4's grid); 600 the round-1 cluster CG with x, r in
# global scratch (grids past 16 warps per row)
@pytest.mark.parametrize("nx", [1, 7, 31, 63, 127, 200, 255, 300, 511, 600])
def test_heat2d_phi_matches_oracle(nx):
    app, hier, cfg, orc = _pair(nx, 65, 1.0, [16], 4, substeps=2)
    drv = T.CycleDriver(app, hier, cfg)
    xs = np.stack([O.random_state(70 + j, nx * nx) for j in range(2)])
    for level in (0, 1):
        got = drv.apply_phi(level, 1, xs)
        for j in range(xs.shape[0]):
            want = orc.step(level, 1 + j, xs[j])
            assert rel_l2(got[j], want) <= 1e-10, (level, j, rel_l2(got[j], want))


@pytest.mark.parametrize("nx", [15, 127])
def test_heat2d_forcing_matches_oracle(nx):
    app, hier, cfg, orc = _pair(nx, 65, 1.0, [16], 4)
    drv = T.CycleDriver(app, hier, cfg)
    got = drv.forcing(0, 1, 3)
    for j in range(3):
        assert rel_l2(got[j], orc.forcing(0, 1 + j)) <= 1e-10


def test_heat2d_symmetry():
    # the stencil commutes with the grid transpose
    nx = 63
    app, hier, cfg, _ = _pair(nx, 65, 1.0, [16], 4, source=False)
    drv = T.CycleDriver(app, hier, cfg)
    x = O.random_state(5, nx * nx)
    xt = x.reshape(nx, nx).T.ravel().copy()
    got = drv.apply_phi(0, 1, np.stack([x, xt]))
    assert rel_l2(got[0].reshape(nx, nx).T.ravel(), got[1]) <= 1e-12


def test_heat2d_config2_shape_two_level():
    # config 2 (two-level, m = 16, k = 4, explicit Gaussian source, u0 = 0)
    # at nx = 31, N_t = 256
    app, hier, cfg, orc = _pair(31, 257, 1.0 / 16, [16], 4, tol=1e-10)
    res = T.solve(app, hier, cfg)
    ref = orc.drive()
    assert res.report.iterations == ref["iterations"], (res.report.iterations, ref["iterations"])
    hist = np.array(res.report.residual_norms)
    assert np.all(np.abs(hist - ref["history"]) <= 1e-8 * np.abs(ref["history"]) + 1e-13)
    assert rel_l2(res.state, orc.array(0)) <= 1e-10


def test_heat2d_config2_grid_short_horizon():
    # config 2's grid (nx = 127, 4-CTA strip cluster) over N_t = 64
    app, hier, cfg, orc = _pair(127, 65, 1.0 / 64, [16], 4, tol=1e-10)
    res = T.solve(app, hier, cfg)
    ref = orc.drive()
    assert res.report.iterations == ref["iterations"]
    assert rel_l2(res.state, orc.array(0)) <= 1e-10


def test_heat2d_config4_shape_fas():
    # config 4 (four-level FAS V-cycle, m = (8, 8, 8), k = 2, folded, smooth
    # Fourier u0) at nx = 31, N_t = 512 over [0, 1/32]
    app, hier, cfg, orc = _pair(31, 513, 1.0 / 32, [8, 8, 8], 2, mode="v-cycle", folded=True,
                                source=False, ic="fourier", tol=1e-10)
    res = T.solve(app, hier, cfg)
    ref = orc.drive()
    assert res.report.iterations == ref["iterations"], (res.report.iterations, ref["iterations"])
    assert rel_l2(res.state, orc.array(0)) <= 1e-10


def test_heat2d_folded_source_nested_fcf():
    app, hier, cfg, orc = _pair(15, 129, 0.25, [4, 4], 3, mode="nested-v", folded=True,
                                relax="FCF", substeps=2, tol=1e-10)
    res = T.solve(app, hier, cfg)
    ref = orc.drive()
    assert res.report.iterations == ref["iterations"]
    assert rel_l2(res.state, orc.array(0)) <= 1e-10


def test_heat2d_cg_cap_raises():
    app, hier, cfg, _ = _pair(31, 65, 1.0, [16], 4, cg_max=2)
    drv = T.CycleDriver(app, hier, cfg)
    with pytest.raises(T.NonlinearSolveError):
        drv.apply_phi(1, 1, O.random_state(1, 31 * 31)[None, :])


def test_heat2d_config4_grid_cluster11_cycles():
    # config 4's grid (nx = 511: group mode, 37 CTAs per system): two cycles
    # incl. the fused C-point norm (group-summed squares) against the
    # oracle's cycles and full residual norm
    app, hier, cfg, orc = _pair(511, 9, 0.01, [4], 2, source=False, ic="fourier", max_iters=2)
    drv = T.CycleDriver(app, hier, cfg)
    drv.setup()
    orc.setup()
    r0 = orc.residual_norm()
    for _ in range(2):
        got = drv.iterate(1)[0]
        orc.cycle()
        want = orc.residual_norm()
        # the second cycle is at rounding level (k = 2 is exact after 2 cycles)
        assert abs(got - want) <= 1e-9 * abs(want) + 1e-12 * r0
    assert rel_l2(drv.get_level(0), orc.array(0)) <= 1e-10


def test_heat2d_inner_iteration_counter():
    # DOF x CG-iterations unit; one Phi = one CG solve whose
    # iterations the counter adds up (0 for families without an inner solve)
    app, hier, cfg, _ = _pair(31, 33, 1.0, [4], 2)
    drv = T.CycleDriver(app, hier, cfg)
    assert drv.inner_iterations() == 0
    x = np.random.default_rng(0).standard_normal((3, 31 * 31))
    drv.apply_phi(0, 1, x[:1])
    one = drv.inner_iterations()
    assert 1 <= one <= 10000
    drv.apply_phi(0, 1, np.repeat(x[:1], 3, axis=0))
    assert drv.inner_iterations() == 4 * one  # identical systems, identical CG runs
    h = T.CycleDriver(T.Heat1D(63), T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, 33), [4], 2),
                      T.SolverConfig())
    h.setup()
    h.iterate(1)
    assert h.inner_iterations() == 0


@pytest.mark.parametrize("nx,npts", [(127, 65), (300, 17)])
def test_strip_cg_solves_are_bitwise_repeatable_and_shard_independent(nx, npts):
    # the strip CG exchanges through DSMEM st.async + mbarriers (127: 4-CTA
    # clusters) or global memory + a release/acquire counter (300: group
    # mode); compute-sanitizer is unavailable on this pool, so races would
    # show here as run-to-run or shard-count differences (the dot products
    # are summed in one fixed order, so every run must be bitwise identical)
    app, hier, cfg, orc = _pair(nx, npts, 1.0 / 64, [4], 2, tol=1e-10, max_iters=6)
    runs = [T.solve(app, hier, cfg) for _ in range(2)] + [T.run_parallel(app, hier, cfg, 3)]
    for r in runs[1:]:
        assert r.report.iterations == runs[0].report.iterations
        assert np.array_equal(np.array(r.report.residual_norms), np.array(runs[0].report.residual_norms))
        assert np.array_equal(r.state, runs[0].state)
    ref = orc.drive()
    assert runs[0].report.iterations == ref["iterations"]
    assert rel_l2(runs[0].state, orc.array(0)) <= 1e-10
