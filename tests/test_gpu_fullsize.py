"""BASELINE configs 2 and 3 at their FULL sizes, and config 4's grid and
four-level hierarchy over a short horizon, against fixtures written by the
compiled reference's own cycle driver (tests/golden/make_fullsize.py:
tempo_ref run_parallel with the restated Phi as its Application): 2D heat
127^2, N_t = 4096, two-level m = 16, k = 4 (CG Phi); Allen-Cahn n = 4096,
N_t = 16384 over [0, 8], three-level m = (8, 8), k = 4 (Newton Phi, FAS
V-cycle); 2D heat 511^2, dt = 4/65536, N_t = 2048, four-level FAS m = (8, 8,
8), k = 2.  All to tol 1e-10 from the seeded random guess.  The bar (BASELINE north star): the
same iteration count, and the final state within 1e-10 relative l2 -- here on
every SAMPLE-th level-0 row the fixture keeps, plus the full state's 2-norm.
The residual histories agree to 1e-8 relative (their tails sit near the
rounding floor of the stopping norm; for the CG Phi of configs 2 and 4 near
its truncation floor, so they are compared absolutely below tol / 4)."""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

import paper_2107_09596_b200 as T
from helpers import rel_l2

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _fixture(tag):
    with open(os.path.join(GOLDEN, f"fullsize_{tag}.json")) as f:
        meta = json.load(f)
    rows = os.path.join(GOLDEN, f"fullsize_{tag}_rows.npy")
    return meta, (np.load(rows) if os.path.exists(rows) else None)


def _objects(c, tol, guess="random", newton_tol=1e-12, meta=None):
    if c == 4:
        app = T.Heat2D(511, folded=True, source=None, cg_rtol=1e-12, cg_max=100000,
                       initial_condition=T.fourier_ic(511))
        hier = T.build_hierarchy(T.TimeGrid.make(0.0, meta["tf"], meta["n_points"]), [8, 8, 8], 2)
        cfg = T.SolverConfig(mode=T.CycleMode.VCycle, relaxation=T.Relaxation.F, max_iters=60,
                             tol=tol, initial_guess=T.InitialGuess.Random, seed=20)
        return app, hier, cfg
    if c == 2:
        app = T.Heat2D(127, folded=False, source=T.gaussian_source(127), cg_rtol=1e-12, cg_max=10000)
        hier = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, 4097), [16], 4)
        mode = T.CycleMode.TwoLevel
    else:
        app = T.AllenCahn(4096, 0.02, 1.0, newton_tol, 30,
                          initial_condition=0.05 * T.random_state(3, 4096))
        hier = T.build_hierarchy(T.TimeGrid.make(0.0, 8.0, 16385), [8, 8], 4)
        mode = T.CycleMode.VCycle
    cfg = T.SolverConfig(mode=mode, relaxation=T.Relaxation.F, max_iters=200, tol=tol,
                         initial_guess=T.InitialGuess.Random if guess == "random" else T.InitialGuess.Constant,
                         seed=20)
    return app, hier, cfg


TAGS = sorted(f[len("fullsize_"):-len(".json")] for f in os.listdir(GOLDEN)
              if f.startswith("fullsize_") and f.endswith(".json"))


@pytest.mark.parametrize("tag", TAGS)
def test_full_size_config_matches_oracle(tag):
    meta, rows = _fixture(tag)
    app, hier, cfg = _objects(meta["config"], meta["tol"], meta.get("guess", "random"),
                              meta.get("newton_tol", 1e-12), meta)
    if "failed_at_iteration" in meta:
        # the oracle's Newton hit its cap (NonlinearSolveError, gray_scott.cpp:
        # 165-169): the device must fail in the same cycle, after the same history
        drv = T.CycleDriver(app, hier, cfg)
        drv.setup()
        hist = []
        with pytest.raises(T.NonlinearSolveError):
            while len(hist) < meta["failed_at_iteration"]:
                hist.append(float(drv.iterate(1)[0]))
        assert len(hist) + 1 == meta["failed_at_iteration"], (len(hist) + 1, meta["failed_at_iteration"])
        ref = np.array(meta["history"])
        assert np.all(np.abs(np.array(hist) - ref) <= 1e-8 * np.abs(ref) + 1e-13)
        return
    res = T.solve(app, hier, cfg)
    assert res.report.converged and meta["converged"]
    assert res.report.iterations == meta["iterations"], (res.report.iterations, meta["iterations"])
    hist = np.array(res.report.residual_norms)
    ref = np.array(meta["history"])
    # 2D heat: each Phi is a CG solve to rtol 1e-12, and the device's
    # Chronopoulos-Gear CG stops at a different iterate than the reference's
    # CG near that threshold; the norms then differ by that truncation
    # (observed <= 2e-11 at the 1e-10 tail), so below a quarter of the
    # stopping tolerance they are compared absolutely
    floor = 0.25 * meta["tol"] if meta["config"] in (2, 4) else 1e-13
    assert np.all(np.abs(hist - ref) <= 1e-8 * np.abs(ref) + floor), np.max(np.abs(hist - ref) / ref)
    got = res.state[::meta["sample_every"], ::meta.get("dof_stride", 1)]
    assert got.shape == rows.shape
    assert rel_l2(got, rows) <= 1e-10, rel_l2(got, rows)
    full = float(np.linalg.norm(res.state))
    assert abs(full - meta["state_l2"]) <= 1e-10 * meta["state_l2"]
