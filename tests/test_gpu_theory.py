"""Solver-theory linkage: the GPU two-level cycle on a
scalar problem propagates the error exactly by the assembled approximate
error propagator E_a (reference test: tests/test_solver.cpp:135-169; E_a:
src/theory.cpp:64-108 error_propagator_approx, restated here for scalars
with numpy instead of Eigen)."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2107_09596_b200 as T

pytestmark = pytest.mark.gpu


def error_propagator_approx(phi: float, psi: float, m: int, k: int, n_t: int) -> np.ndarray:
    """(N_t+1)x(N_t+1) E_a of the truncated two-level cycle: block row of
    coarse point p (fine rows p m + a, a < m) receives, from coarse column
    p - d (d = 1..min(k, p)), phi^a * payload_d with payload_d =
    psi^(d-1) (phi^m - psi) for d < k and psi^(k-1) phi^m for d = k."""
    E = np.zeros((n_t + 1, n_t + 1))
    defect = phi ** m - psi
    payload = {d: psi ** (d - 1) * defect for d in range(1, k)}
    payload[k] = psi ** (k - 1) * phi ** m
    n_blocks = n_t // m + 1
    for p in range(1, n_blocks):
        row_c = p * m
        height = min(m, n_t + 1 - row_c)
        for d in range(1, min(k, p) + 1):
            col = (p - d) * m
            for a in range(height):
                E[row_c + a, col] = phi ** a * payload[d]
    return E


@pytest.mark.parametrize("phi,psi,n_t,m,k,seed", [
    (0.5, 0.3, 4, 2, 2, 31),       # the reference test's case
    (0.9, 0.6, 32, 4, 3, 7),
    (0.95, 0.5, 64, 8, 2, 11),
    (0.8, 0.7, 30, 4, 4, 3),       # short trailing interval
])
def test_cycle_error_follows_error_propagator(phi, psi, n_t, m, k, seed):
    n_points = n_t + 1
    app = T.ScalarLinear([phi, psi], 1.0, False)
    hier = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, n_points), [m], k)
    cfg = T.SolverConfig(mode=T.CycleMode.TwoLevel, initial_guess=T.InitialGuess.Random, seed=seed,
                         tol=1e-300, max_iters=5)
    exact = phi ** np.arange(n_points)  # sequential solution u_i = phi u_{i-1}, u_0 = 1
    Ea = error_propagator_approx(phi, psi, m, k, n_t)
    drv = T.CycleDriver(app, hier, cfg)
    drv.setup()
    err = drv.get_level(0)[:, 0] - exact
    for _ in range(5):
        drv.cycle()
        predicted = Ea @ err
        err = drv.get_level(0)[:, 0] - exact
        scale = max(np.max(np.abs(predicted)), 1e-300)
        assert np.max(np.abs(err - predicted)) <= 1e-12 * scale + 1e-15, (err, predicted)


def error_propagator_approx_blocks(Phi: np.ndarray, Psi: np.ndarray, m: int, k: int, n_t: int):
    """Block version (n x n blocks) of error_propagator_approx."""
    n = Phi.shape[0]
    E = np.zeros(((n_t + 1) * n, (n_t + 1) * n))
    P = [np.linalg.matrix_power(Phi, a) for a in range(m + 1)]
    defect = P[m] - Psi
    payload = {d: np.linalg.matrix_power(Psi, d - 1) @ defect for d in range(1, k)}
    payload[k] = np.linalg.matrix_power(Psi, k - 1) @ P[m]
    for p in range(1, n_t // m + 1):
        row_c = p * m
        for d in range(1, min(k, p) + 1):
            col = (p - d) * m
            for a in range(min(m, n_t + 1 - row_c)):
                r = (row_c + a) * n
                E[r:r + n, col * n:col * n + n] = P[a] @ payload[d]
    return E


@pytest.mark.parametrize("n,n_t,m,k", [(7, 16, 4, 2), (15, 24, 4, 3)])
def test_heat_cycle_error_follows_block_error_propagator(n, n_t, m, k):
    # heat1d (homogeneous): Phi = (I + dt L)^-1, Psi = (I + m dt L)^-1, dense
    app = T.Heat1D(n, manufactured_forcing=False)
    hier = T.build_hierarchy(T.TimeGrid.make(0.0, 0.5, n_t + 1), [m], k)
    cfg = T.SolverConfig(mode=T.CycleMode.TwoLevel, initial_guess=T.InitialGuess.Random, seed=9,
                         tol=1e-300, max_iters=4)
    h = 1.0 / (n + 1)
    Lap = (2 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)) / (h * h)
    dt = 0.5 / n_t
    Phi = np.linalg.inv(np.eye(n) + dt * Lap)
    Psi = np.linalg.inv(np.eye(n) + m * dt * Lap)
    u0 = np.sin(np.pi * h * np.arange(1, n + 1))
    exact = np.stack([np.linalg.matrix_power(Phi, i) @ u0 for i in range(n_t + 1)]).ravel()
    Ea = error_propagator_approx_blocks(Phi, Psi, m, k, n_t)
    drv = T.CycleDriver(app, hier, cfg)
    drv.setup()
    err = drv.get_level(0).ravel() - exact
    for _ in range(4):
        drv.cycle()
        predicted = Ea @ err
        err = drv.get_level(0).ravel() - exact
        assert np.max(np.abs(err - predicted)) <= 1e-11 * max(np.max(np.abs(predicted)), 1e-14) + 1e-14
