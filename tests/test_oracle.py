"""CPU: pin the oracle restatement (oracle/atm_oracle.c).

1. The reference's own known-answer tests and oracle properties, restated
   without doctest/Eigen (tests/test_kernels.cpp, tests/test_solver.cpp,
   tests/support.hpp of /root/reference/proj).
2. Bitwise agreement with the committed fixtures produced by the compiled
   reference (tests/golden/make_golden.py -> oracle/_ref/tempo_ref).
3. Where the compiled reference is present, bitwise agreement on fresh runs.
"""
import math

import numpy as np
import pytest

from conftest import golden_array, golden_cases
from helpers import oracle_driver
from oracle import oracle as O


def scalar(mult, n_points, m, k=2, ff=None, folded=0, **solver):
    return O.Driver(dict(kind=O.SCALAR, mult=mult, u0=1.0, folded=folded, fine_forcing=ff),
                    dict(tf=1.0, n_points=n_points, m=m, k=k), solver)


# ---------------------------------------------------------------- splitmix64

def test_random_state_deterministic_and_in_range():
    # tests/test_core.cpp: determinism, range [-1, 1), seed sensitivity
    a, b = O.random_state(42, 1000), O.random_state(42, 1000)
    assert np.array_equal(a, b)
    assert a.min() >= -1.0 and a.max() < 1.0
    assert not np.array_equal(a, O.random_state(43, 1000))


def test_random_state_matches_python_splitmix():
    def mix(z):
        M = (1 << 64) - 1
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)
    s = 7
    want = []
    for q in range(16):
        s = (s + 0x9E3779B97F4A7C15) & ((1 << 64) - 1)
        want.append(2.0 * ((mix(s) >> 11) * 2.0 ** -53) - 1.0)
    assert np.array_equal(O.random_state(7, 16), np.array(want))


# ------------------------------------------------------- kernel known answers

def test_f_relax_known_answer():
    # test_kernels.cpp:39-47
    d = scalar([0.5, 0.25], 5, 2)
    d.setup()
    u = d.array(0)
    u[:, 0] = [1, 9, 3, 9, 5]
    d.array(1 - 1, "g")[:, 0] = 0.0
    d.f_relax(0, 0, 2)
    assert u[:, 0].tolist() == [1, 0.5, 3, 1.5, 5]


def test_c_then_f_relax_known_answer():
    # test_kernels.cpp:86-96
    d = scalar([0.5, 0.25], 5, 2)
    d.setup()
    u = d.array(0)
    u[:, 0] = [1, 0.5, 3, 1.5, 5]
    d.array(0, "g")[:, 0] = 0.0
    d.c_relax(0, 0, 3)
    assert u[:, 0].tolist() == [1, 0.5, 0.25, 1.5, 0.75]
    d.f_relax(0, 0, 2)
    assert u[:, 0].tolist() == [1, 0.5, 0.25, 0.125, 0.75]


def test_zero_integrator_leaves_forcing():
    # test_kernels.cpp:49-57
    d = scalar([0.0, 0.0], 5, 2)
    d.setup()
    d.array(0)[:, 0] = [4, 7, -2, 9, 3]
    d.array(0, "g")[:, 0] = 1.0
    d.f_relax(0, 0, 2)
    assert d.array(0)[:, 0].tolist() == [4, 1, -2, 1, 3]


def test_residual_known_answer():
    # test_kernels.cpp:141-149
    d = scalar([0.5, 0.25], 3, 2)
    d.setup()
    d.array(0)[:, 0] = [1, 0, 0]
    g = d.array(0, "g")
    g[:, 0] = [1, 0, 0]
    assert d.residual(0, 0, 3)[:, 0].tolist() == [0, 0.5, 0]


def test_untruncated_window_equals_forward_solve():
    # test_kernels.cpp:183-203
    phi, psi, nc = 0.6, 0.35, 7
    d = scalar([phi, psi], 13, 2, k=nc)
    r = np.stack([O.random_state(7 + j, 1) for j in range(nc)])
    e = np.zeros(nc)
    e[0] = r[0, 0]
    for j in range(1, nc):
        e[j] = psi * e[j - 1] + r[j, 0]
    for p in range(nc):
        got = d.window_linear(1, 0, r[: p + 1])[0]
        assert got == pytest.approx(e[p], rel=1e-14)


def test_k1_windows_and_fas_equals_linear():
    # test_kernels.cpp:205-233
    d = scalar([0.5, 0.25], 9, 2)
    r = O.random_state(3, 1)[None, :]
    assert d.window_linear(1, 4, r)[0] == r[0, 0]
    v = O.random_state(4, 1)[None, :]
    assert d.window_fas(1, 4, v, r)[0] == v[0, 0] + r[0, 0]
    d2 = scalar([0.8, 0.61], 17, 2, k=4)
    vv = np.stack([O.random_state(40 + j, 1) for j in range(4)])
    rr = np.stack([O.random_state(50 + j, 1) for j in range(4)])
    un = d2.window_fas(1, 2, vv, rr)[0]
    e = d2.window_linear(1, 2, rr)[0]
    assert un - vv[3, 0] == pytest.approx(e, rel=1e-13)


# --------------------------------------------------------- solver properties

def _dahl(n_points, tf, m, k, **s):
    return O.Driver(dict(kind=O.DAHLQUIST, lam=-1.0, u0=1.0, folded=s.pop("folded", 0)),
                    dict(tf=tf, n_points=n_points, m=m, k=k), s)


def test_exact_after_nt_iterations_for_every_k():
    # test_solver.cpp:81-103
    mult = 1.0 / (1.0 + 4.0 / 64)
    exact = np.array([mult ** i for i in range(65)])
    for k in range(2, 10):
        d = _dahl(65, 4.0, 8, k, initial_guess=O.GUESS_RANDOM, seed=99, tol=1e-300, max_iters=8)
        d.setup()
        for _ in range(8):
            d.cycle()
        assert np.max(np.abs(d.array(0)[:, 0] - exact)) < 1e-12


def _parareal(phi, psi, n_points, m, guess, iters):
    """tests/support.hpp:80-172 restated (scalar)."""
    nc = (n_points - 1) // m + 1
    U = [guess[j * m] for j in range(nc)]
    U[0] = 1.0
    hist = []
    for _ in range(iters):
        fine = [0.0] * nc
        for j in range(1, nc):
            u = U[j - 1]
            for _i in range(m):
                u = phi * u
            fine[j] = u
        nxt = [1.0] + [0.0] * (nc - 1)
        for j in range(1, nc):
            nxt[j] = psi * nxt[j - 1] + fine[j] - psi * U[j - 1]
        U = nxt
        u = np.zeros(n_points)
        for j in range(nc):
            u[j * m] = U[j]
        for j in range(nc):
            for i in range(j * m + 1, min(j * m + m, n_points)):
                u[i] = phi * u[i - 1]
        res = [1.0 - u[0]] + [phi * u[i - 1] - u[i] for i in range(1, n_points)]
        hist.append(math.sqrt(sum(x * x for x in res)))
    return hist


def test_global_window_reproduces_parareal():
    # test_solver.cpp:105-133
    guess = np.concatenate([[1.0], [O.random_state(7 + i, 1)[0] for i in range(1, 33)]])
    d = _dahl(33, 2.0, 4, 9, initial_guess=O.GUESS_PROVIDED, provided=guess, tol=1e-300, max_iters=8)
    got = d.drive()["history"]
    phi = 1.0 / (1.0 + 2.0 / 32)
    psi = 1.0 / (1.0 + 4 * 2.0 / 32)
    want = _parareal(phi, psi, 33, 4, guess, 8)
    for a, b in zip(got, want):
        assert a == pytest.approx(b, rel=1e-12, abs=1e-12 * want[0])


def test_two_level_fas_equals_linear_correction():
    # test_solver.cpp:171-204
    lin = _dahl(33, 2.0, 4, 3, initial_guess=O.GUESS_RANDOM, seed=5, tol=1e-300)
    fas = _dahl(33, 2.0, 4, 3, folded=1, mode=O.VCYCLE, initial_guess=O.GUESS_RANDOM, seed=5,
                tol=1e-300)
    lin.setup()
    fas.setup()
    for _ in range(4):
        lin.cycle()
        fas.cycle()
        assert np.allclose(lin.array(0), fas.array(0), rtol=1e-12, atol=0)


def test_exact_solution_is_a_fixed_point():
    # test_solver.cpp:243-282
    ff = np.array([0.0] + [math.sin(0.37 * i) for i in range(1, 33)])
    for k in (2, 4, 9):
        for folded, mode in ((0, O.TWO_LEVEL), (1, O.VCYCLE)):
            seq = np.zeros(33)
            seq[0] = 1.0
            for i in range(1, 33):
                seq[i] = 0.6 * seq[i - 1] + ff[i]
            d = scalar([0.6, 0.36], 33, 4, k=k, ff=ff, folded=folded, mode=mode,
                       initial_guess=O.GUESS_PROVIDED, provided=seq, tol=1e-300)
            d.grid  # noqa
            d.setup()
            d.cycle()
            assert np.max(np.abs(d.array(0)[:, 0] - seq)) < 1e-13


def test_front_advances_k_points_per_iteration():
    # test_solver.cpp:428-465 (ceil(N_T / k))
    for nt, k in ((6, 2), (6, 3), (8, 2), (8, 4), (12, 3)):
        n_points = 2 * (nt + 1)
        d = _dahl(n_points, 1.0, 2, k, initial_guess=O.GUESS_CONSTANT,
                  constant_value=np.zeros(1), tol=1e-300)
        d.setup()
        it = 0
        while np.any(d.array(0)[::2, 0] == 0.0) and it < 100:
            d.cycle()
            it += 1
        assert it == (nt + k - 1) // k


def test_fcf_not_slower_than_f():
    # test_solver.cpp:284-300
    its = {}
    for relax in (O.RELAX_F, O.RELAX_FCF):
        d = _dahl(65, 2.0, 8, 3, relaxation=relax, initial_guess=O.GUESS_RANDOM, seed=3,
                  tol=1e-10, max_iters=50)
        its[relax] = d.drive()["iterations"]
    assert its[O.RELAX_FCF] <= its[O.RELAX_F]


def test_nested_iterations_known_answer():
    # test_solver.cpp:302-331
    d = _dahl(17, 2.0, 4, 5, folded=1, mode=O.NESTED_V, tol=1e-300)
    d.setup()
    d.nested_init()
    psi = 1.0 / (1.0 + 0.5)
    phi = 1.0 / (1.0 + 0.125)
    coarse = [psi ** j for j in range(5)]
    want = [coarse[i // 4] * phi ** (i % 4) for i in range(17)]
    assert np.allclose(d.array(0)[:, 0], want, rtol=1e-13)


def test_divergence_and_config_errors():
    # test_solver.cpp:391-425
    d = O.Driver(dict(kind=O.DAHLQUIST, lam=1.0, u0=1.0), dict(tf=32.0, n_points=33, m=4, k=3),
                 dict(initial_guess=O.GUESS_RANDOM, tol=1e-7))
    with pytest.raises(O.OracleError) as ei:
        d.drive()
    assert ei.value.code == O.ORC_DIVERGED if hasattr(O, "ORC_DIVERGED") else ei.value.code == 4
    with pytest.raises(O.OracleError):
        O.Driver(dict(kind=O.DAHLQUIST, folded=1), dict(tf=2.0, n_points=33, m=4, k=3), dict())
    with pytest.raises(O.OracleError):
        O.Driver(dict(kind=O.DAHLQUIST, folded=0), dict(tf=2.0, n_points=33, m=4, k=3),
                 dict(mode=O.VCYCLE))


def test_huge_tolerance_single_iteration():
    d = _dahl(33, 2.0, 4, 3, initial_guess=O.GUESS_RANDOM, tol=1e6)
    r = d.drive()
    assert r["converged"] and r["iterations"] == 1


def test_heat_residual_of_sequential_solution_is_zero():
    d = O.Driver(dict(kind=O.HEAT1D, n=17), dict(tf=1.0, n_points=9, m=4, k=2), dict())
    d.setup()
    u = d.array(0)
    g = d.array(0, "g")
    for i in range(1, 9):
        u[i] = d.step(0, i, u[i - 1]) + g[i]
    assert np.all(d.residual(0, 0, 9) == 0.0)


# --------------------------------------------------------- golden fixtures

FAST = ["config1", "dahlquist_cfg", "heat_det_65", "heat_fas_nested_fcf", "heat_fas_vcycle_f"]


@pytest.mark.parametrize("name", FAST)
def test_oracle_bitwise_equals_compiled_reference_fixture(name):
    case = golden_cases()[name]
    ic = golden_array(name, "ic") if case.get("has_ic") else None
    d = oracle_driver(case["args"], ic=ic)
    r = d.drive()
    assert r["iterations"] == case["iterations"]
    assert r["history"].tolist() == case["history"]
    if case.get("store_u"):
        assert np.array_equal(d.array(0), golden_array(name, "u"))


@pytest.mark.slow
@pytest.mark.parametrize("name", ["heat_full_single", "kstudy_k2", "kstudy_k128"])
def test_oracle_matches_reference_heat_study(name):
    case = golden_cases()[name]
    d = oracle_driver(case["args"])
    r = d.drive()
    assert r["iterations"] == case["iterations"]
    assert r["history"].tolist() == case["history"]


@pytest.mark.skipif(not O.ref_available(), reason="compiled reference not built here")
def test_oracle_equals_fresh_reference_run():
    args = dict(problem="heat1d", n=33, tf=2.0, n_points=129, m="4,4", k=3, folded=1,
                mode="nested-v", relax="FCF", guess="random", seed=11, tol=1e-9, max_iters=30,
                substeps=2)
    res, u = O.run_ref(dict(args, workers=1), out_u=True)
    d = oracle_driver(args)
    r = d.drive()
    assert r["history"].tolist() == res["history"]
    assert np.array_equal(d.array(0).reshape(-1), u)


# The reference has no Phi for configs 2-4 / Gray-Scott; tempo_ref's OracleApp
# runs the restated Phi (ac_step, h2_solve, gs_step) inside the reference's
# own CycleDriver (solver.cpp:152-435) over run_parallel's worker threads.
# The oracle's own cycle restatement must agree with it bitwise on the shapes
# of BASELINE configs 2, 3, 4 (reduced) and the Gray-Scott desk problem.
def _ref_small_cases():
    import paper_2107_09596_b200 as T
    nx2, n3, nx4 = 15, 64, 31
    src = T.gaussian_source(nx2)
    ic3 = 0.05 * O.random_state(3, n3)
    ic4 = T.fourier_ic(nx4)
    return {
        "config2_shape": (dict(problem="heat2d", nx=nx2, folded=0, cg_rtol=1e-12, cg_max=10000, tf=1.0,
                               n_points=257, m="16", k=4, mode="two-level", guess="random", seed=20,
                               max_iters=100, tol=1e-10), dict(source_file=src)),
        "config3_shape": (dict(problem="allen_cahn", n=n3, eps=0.02, length=1.0, newton_tol=1e-12,
                               newton_max=30, tf=8.0, n_points=1025, m="8,8", k=4, mode="v-cycle",
                               guess="random", seed=20, max_iters=200, tol=1e-10), dict(ic_file=ic3)),
        "config4_shape": (dict(problem="heat2d", nx=nx4, folded=1, cg_rtol=1e-12, cg_max=100000, tf=0.125,
                               n_points=257, m="4,4,4", k=2, mode="v-cycle", guess="random", seed=20,
                               max_iters=60, tol=1e-10), dict(ic_file=ic4)),
        "grayscott_nested": (dict(problem="gray_scott", nx=16, tf=64.0, n_points=257, m="16", k=8,
                                  mode="nested-v", guess="constant", seed=0, max_iters=60, tol=1e-7), {}),
    }


def _oracle_from_ref_args(args, files):
    kind = {"heat2d": O.HEAT2D, "allen_cahn": O.ALLEN_CAHN, "gray_scott": O.GRAY_SCOTT}[args["problem"]]
    p = dict(kind=kind, folded=args.get("folded", 1))
    if kind == O.HEAT2D:
        nx = args["nx"]
        p.update(n=nx * nx, nx=nx, cg_rtol=args["cg_rtol"], cg_max=args["cg_max"],
                 source=files.get("source_file"), ic=files.get("ic_file"))
    elif kind == O.ALLEN_CAHN:
        p.update(n=args["n"], eps=args["eps"], length=args["length"], newton_tol=args["newton_tol"],
                 newton_max=args["newton_max"], ic=files["ic_file"])
    else:
        p.update(nx=args["nx"], n=2 * args["nx"] ** 2)
    g = dict(tf=args["tf"], n_points=args["n_points"], m=[int(x) for x in str(args["m"]).split(",")],
             k=args["k"])
    mode = {"two-level": O.TWO_LEVEL, "v-cycle": O.VCYCLE, "nested-v": O.NESTED_V}[args["mode"]]
    s = dict(mode=mode, relaxation=O.RELAX_F, max_iters=args["max_iters"], tol=args["tol"],
             initial_guess=O.GUESS_RANDOM if args["guess"] == "random" else O.GUESS_CONSTANT,
             seed=args["seed"])
    return O.Driver(p, g, s)


@pytest.mark.skipif(not O.ref_available(), reason="compiled reference not built here")
@pytest.mark.parametrize("name", ["config2_shape", "config3_shape", "config4_shape", "grayscott_nested"])
def test_oracle_cycles_equal_reference_cycle_driver_on_restated_phi(name):
    args, files = _ref_small_cases()[name]
    res, u = O.run_ref(dict(args, workers=0), out_u=True, files=files)
    assert "error" not in res, res
    d = _oracle_from_ref_args(args, files)
    r = d.drive()
    assert r["iterations"] == res["iterations"] and r["converged"] == res["converged"]
    assert r["history"].tolist() == res["history"]
    assert np.array_equal(d.array(0).reshape(-1), u)
