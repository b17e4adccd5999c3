"""Allen-Cahn (BASELINE config 3) on the device vs the C oracle.

No reference Phi exists for this family: the oracle's
ac_step (oracle/atm_oracle.c) restates backward Euler + exact Newton on the
cyclic tridiagonal Jacobian with the stopping rule of gray_scott.cpp:113.
The device solves the Newton systems by Richardson on the shifted constant
part (heat_phi5.cu ac_phi), so iterates agree to rounding; the bar is the
solver's: same MGRIT iteration count, final u within 1e-10 relative l2.
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_2107_09596_b200 as T
from helpers import rel_l2
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _pair(n, n_points, tf, ms, k, mode="v-cycle", tol=1e-9, max_iters=60, newton_max=30,
          substeps=1, ic_seed=3, guess_seed=20, relax="F"):
    ic = 0.05 * O.random_state(ic_seed, n)
    app = T.AllenCahn(n, 0.02, 1.0, 1e-12, newton_max, initial_condition=ic)
    hier = T.build_hierarchy(T.TimeGrid.make(0.0, tf, n_points), ms, k)
    cm = {"v-cycle": T.CycleMode.VCycle, "nested-v": T.CycleMode.NestedV}[mode]
    cfg = T.SolverConfig(mode=cm, relaxation=T.Relaxation.FCF if relax == "FCF" else T.Relaxation.F,
                         max_iters=max_iters, tol=tol, initial_guess=T.InitialGuess.Random,
                         seed=guess_seed, coarse_substeps=substeps)
    orc = O.Driver(dict(kind=O.ALLEN_CAHN, n=n, eps=0.02, length=1.0, newton_tol=1e-12,
                        newton_max=newton_max, folded=1, ic=ic),
                   dict(tf=tf, n_points=n_points, m=list(ms), k=k),
                   dict(mode={"v-cycle": O.VCYCLE, "nested-v": O.NESTED_V}[mode],
                        relaxation=O.RELAX_FCF if relax == "FCF" else O.RELAX_F,
                        max_iters=max_iters, tol=tol, initial_guess=O.GUESS_RANDOM,
                        seed=guess_seed, coarse_substeps=substeps))
    return app, hier, cfg, orc


@pytest.mark.parametrize("n", [16, 17, 64, 100, 264, 1001, 1024, 4093, 4096])
@pytest.mark.parametrize("level", [0, 1, 2])
def test_ac_phi_matches_oracle(n, level):
    app, hier, cfg, orc = _pair(n, 257, 1.0, [8, 8], 4, substeps=2)
    drv = T.CycleDriver(app, hier, cfg)
    # small-amplitude states (config 3's regime) and full [-1, 1) states
    xs = np.stack([0.05 * O.random_state(50 + j, n) for j in range(2)] +
                  [O.random_state(60 + j, n) for j in range(2)])
    got = drv.apply_phi(level, 1, xs)
    for j in range(xs.shape[0]):
        want = orc.step(level, 1 + j, xs[j])
        assert rel_l2(got[j], want) <= 1e-11, (j, rel_l2(got[j], want))


def test_ac_periodic_wrap_and_symmetry():
    # a shifted input gives the shifted output (periodicity through the
    # Woodbury corners), and -u maps to -Phi(u) (odd nonlinearity)
    n = 512
    app, hier, cfg, _ = _pair(n, 257, 1.0, [8, 8], 4)
    drv = T.CycleDriver(app, hier, cfg)
    x = O.random_state(9, n)
    xs = np.stack([x, np.roll(x, 37), -x])
    got = drv.apply_phi(1, 1, xs)
    assert rel_l2(np.roll(got[0], 37), got[1]) <= 1e-12
    assert rel_l2(-got[0], got[2]) <= 1e-13


@pytest.mark.parametrize("n,n_points,tf,k", [(256, 513, 0.25, 4), (1024, 1025, 0.5, 2), (1001, 513, 0.25, 4)])
def test_ac_fas_vcycle_matches_oracle(n, n_points, tf, k):
    app, hier, cfg, orc = _pair(n, n_points, tf, [8, 8], k)
    res = T.solve(app, hier, cfg)
    ref = orc.drive()
    assert res.report.iterations == ref["iterations"], (res.report.iterations, ref["iterations"])
    assert res.report.converged == ref["converged"]
    hist = np.array(res.report.residual_norms)
    assert np.all(np.abs(hist - ref["history"]) <= 1e-8 * np.abs(ref["history"]) + 1e-12)
    assert rel_l2(res.state, orc.array(0)) <= 1e-10


def test_ac_config3_shape_reduced():
    # config 3 (n = 4096, dt = 1/2048, m = (8, 8), k = 4, FAS V-cycle) at
    # N_t = 1024
    app, hier, cfg, orc = _pair(4096, 1025, 0.5, [8, 8], 4, tol=1e-10)
    res = T.solve(app, hier, cfg)
    ref = orc.drive()
    assert res.report.iterations == ref["iterations"], (res.report.iterations, ref["iterations"])
    assert rel_l2(res.state, orc.array(0)) <= 1e-10


def test_ac_nested_fcf_substeps_matches_oracle():
    app, hier, cfg, orc = _pair(128, 257, 0.5, [4, 4], 3, mode="nested-v", relax="FCF", substeps=2)
    res = T.solve(app, hier, cfg)
    ref = orc.drive()
    assert res.report.iterations == ref["iterations"]
    assert rel_l2(res.state, orc.array(0)) <= 1e-10


def test_ac_newton_cap_raises():
    # one Newton iteration cannot reach 1e-12 from a [-1, 1) guess
    app, hier, cfg, _ = _pair(64, 65, 1.0, [8, 8], 2, newton_max=1)
    drv = T.CycleDriver(app, hier, cfg)
    with pytest.raises(T.NonlinearSolveError):
        drv.apply_phi(0, 1, O.random_state(1, 64)[None, :])


def test_ac_and_heat_fas_cycles_are_deterministic():
    # repeated runs are bitwise identical (guards the staging-buffer hazards
    # of the FAS sweeps with stored right-hand sides)
    app, hier, cfg, _ = _pair(4096, 2049, 1.0, [8, 8], 4)
    runs = []
    for _ in range(3):
        d = T.CycleDriver(app, hier, cfg)
        d.setup()
        norms = d.iterate(2)
        runs.append((norms, d.get_level(0)))
    for norms, u in runs[1:]:
        assert np.array_equal(norms, runs[0][0])
        assert np.array_equal(u, runs[0][1])
    heat = T.Heat1D(4095, folded=True, manufactured_forcing=True)
    hh = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, 4097), [8, 8], 4)
    hc = T.SolverConfig(mode=T.CycleMode.VCycle, max_iters=10, tol=1e-12,
                        initial_guess=T.InitialGuess.Random, seed=20)
    hr = []
    for _ in range(3):
        d = T.CycleDriver(heat, hh, hc)
        d.setup()
        hr.append((d.iterate(2), d.get_level(0)))
    for norms, u in hr[1:]:
        assert np.array_equal(norms, hr[0][0])
        assert np.array_equal(u, hr[0][1])
