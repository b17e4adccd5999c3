"""GPU parity: the CUDA path (through the C ABI) against the C oracle
restatement and the compiled-reference fixtures.  Tolerances: Phi and kernel
outputs 1e-12 relative (the device Thomas solve is a blocked scan, so it
rounds differently from the serial reference); solves: identical iteration
count and final solution within 1e-10 relative l2 (BASELINE north star)."""
import math

import numpy as np
import pytest

import paper_2107_09596_b200 as T
from conftest import golden_array, golden_cases
from helpers import device_objects, oracle_driver, rel_l2
from oracle import oracle as O

pytestmark = pytest.mark.gpu

PHI_RTOL = 1e-12
SOLVE_RTOL = 1e-10


def _heat_case(n, n_points=33, m=4, k=3, folded=0, manufactured=0, substeps=1, mode="two-level"):
    return dict(problem="heat1d", n=n, tf=1.0, n_points=n_points, m=m, k=k, folded=folded,
                manufactured=manufactured, substeps=substeps, mode=mode, guess="random", seed=5,
                max_iters=50, tol=1e-9)


def _thomas_ld(n, r, rhs, substeps):
    """Extended-precision (x87 long double) restatement of the reference
    Thomas solve (heat1d.cpp:47-60), the yardstick for both fp64 paths."""
    L = np.longdouble
    r = L(r)
    a, b = -r, L(1) + 2 * r
    cp = np.zeros(n, L)
    inv = np.zeros(n, L)
    prev = L(0)
    for i in range(n):
        den = b - a * prev
        inv[i] = L(1) / den
        prev = a / den
        cp[i] = prev
    x = np.asarray(rhs, L).copy()
    for _ in range(substeps):
        p = L(0)
        for i in range(n):
            p = (x[i] - a * p) * inv[i]
            x[i] = p
        for i in range(n - 2, -1, -1):
            x[i] -= cp[i] * x[i + 1]
    return x


def _check_phi(drv, orc, hier, n, level, first, xs, substeps):
    """Device Phi must be at least as accurate as the reference's own fp64
    Thomas sweep (plus 1e-14 slack), measured against an extended-precision
    solve; and within 1e-11 of the reference itself (or of the sum of both
    errors, when the reference's error alone exceeds that)."""
    got = drv.apply_phi(level, first, xs)
    dt = hier.level(level).dt / substeps
    h = 1.0 / (n + 1)
    r = dt / (h * h)
    for j in range(xs.shape[0]):
        ref = orc.step(level, first + j, xs[j])
        ex = _thomas_ld(n, r, xs[j], substeps)
        scale = float(np.linalg.norm(np.asarray(ex, np.float64)))
        e_dev = float(np.linalg.norm(np.asarray(got[j] - ex, np.float64))) / scale
        e_ref = float(np.linalg.norm(np.asarray(ref - ex, np.float64))) / scale
        assert e_dev <= max(2.0 * e_ref, 1e-14), (e_dev, e_ref)
        # within 1e-11 of the reference, or -- where the reference's own
        # rounding error is larger (stiff rows, large n) -- within the
        # triangle bound of the two errors against the extended-precision solve
        assert rel_l2(got[j], ref) <= max(1e-11, 1.01 * (e_dev + e_ref))


@pytest.mark.parametrize("n", [1, 2, 17, 63, 64, 65, 257, 1025, 2049, 4095, 4096, 4097, 5000, 5375, 5376, 5377, 8191, 12289, 16384, 40001])
@pytest.mark.parametrize("level", [0, 1])
def test_phi_matches_oracle(n, level):
    args = _heat_case(n, substeps=3)
    app, hier, cfg = device_objects(args)
    drv = T.CycleDriver(app, hier, cfg)
    orc = oracle_driver(args)
    xs = np.stack([O.random_state(100 + j, n) for j in range(3)])
    _check_phi(drv, orc, hier, n, level, 1, xs, 3 if level == 1 else 1)


@pytest.mark.parametrize("n", [33, 100, 1000, 2051, 2053, 2056, 3003, 4090])
def test_phi_sub_block_solver_matches_oracle(n, monkeypatch):
    # ATM_HEAT_L=16 puts every level on the L = 16 kernels, i.e. the
    # sub-block solve (tri_solve_sb): row ends at every position of a chunk's
    # two 8-element sub-blocks (n % 16 = 1, 4, 8, 3, 5, 8, 11, 10), rows of one
    # to 257 chunks, three sub-steps
    monkeypatch.setenv("ATM_HEAT_L", "16")
    args = _heat_case(n, substeps=3)
    app, hier, cfg = device_objects(args)
    drv = T.CycleDriver(app, hier, cfg)
    orc = oracle_driver(args)
    xs = np.stack([O.random_state(100 + j, n) for j in range(3)])
    for level in (0, 1):
        _check_phi(drv, orc, hier, n, level, 1, xs, 3 if level == 1 else 1)


@pytest.mark.parametrize("n", [2053, 4090, 4096])
@pytest.mark.parametrize("tf", [1e-9, 1e-4, 64.0])
def test_phi_sub_block_solver_across_stiffness(n, tf, monkeypatch):
    # dt/h^2 from ~1e-4 (gamma^8 ~ 1e-33: the kappa of a short sub-block is a
    # large number times a tiny p_b) to ~1e7 (carries reach across the row)
    monkeypatch.setenv("ATM_HEAT_L", "16")
    args = dict(_heat_case(n, n_points=4097, m=16, k=8), tf=tf)
    app, hier, cfg = device_objects(args)
    drv = T.CycleDriver(app, hier, cfg)
    orc = oracle_driver(args)
    xs = np.stack([O.random_state(300 + j, n) for j in range(2)])
    for level in (0, 1):
        _check_phi(drv, orc, hier, n, level, 1, xs, 1)


@pytest.mark.parametrize("n", [63, 257, 1025, 4095])
@pytest.mark.parametrize("tf", [1.0 / 64, 1.0 / 4, 4.0])
def test_phi_across_stiffness(n, tf):
    # dt/h^2 from O(1) to O(1e5): the Sherman-Morrison boundary correction
    # spans one warp to the whole vector
    args = dict(_heat_case(n, n_points=4097, m=16, k=8), tf=tf)
    app, hier, cfg = device_objects(args)
    drv = T.CycleDriver(app, hier, cfg)
    orc = oracle_driver(args)
    xs = np.stack([O.random_state(300 + j, n) for j in range(2)])
    for level in (0, 1):
        _check_phi(drv, orc, hier, n, level, 1, xs, 1)


@pytest.mark.parametrize("n", [17, 1025])
def test_forced_phi_and_forcing_match_oracle(n):
    for folded in (0, 1):
        args = _heat_case(n, folded=folded, manufactured=1, substeps=2,
                          mode="two-level" if not folded else "v-cycle")
        app, hier, cfg = device_objects(args)
        drv = T.CycleDriver(app, hier, cfg)
        orc = oracle_driver(args)
        x = np.stack([O.random_state(7 + j, n) for j in range(4)])
        got = drv.apply_phi(1, 3, x)
        want = np.stack([orc.step(1, 3 + j, x[j]) for j in range(4)])
        assert rel_l2(got, want) <= PHI_RTOL
        gf = drv.forcing(0, 1, 6)
        wf = np.stack([orc.forcing(0, 1 + j) for j in range(6)])
        assert rel_l2(gf, wf) <= PHI_RTOL


def test_f_relax_c_relax_residual_kernels():
    n = 129
    args = _heat_case(n, n_points=49, m=6, manufactured=1)
    app, hier, cfg = device_objects(args)
    drv = T.CycleDriver(app, hier, cfg)
    drv.setup()
    orc = oracle_driver(args)
    orc.setup()
    u0 = drv.get_level(0)
    assert np.array_equal(u0, orc.array(0)), "device random fill must be bitwise the reference's"
    split = hier.split(0)
    drv.f_relax(0, 0, len(split.intervals))
    orc.f_relax(0, 0, len(split.intervals))
    assert rel_l2(drv.get_level(0), orc.array(0)) <= PHI_RTOL
    drv.c_relax(0, 0, len(split.c_points))
    orc.c_relax(0, 0, len(split.c_points))
    assert rel_l2(drv.get_level(0), orc.array(0)) <= PHI_RTOL
    r_dev = drv.residual(0, 0, 49)
    r_orc = orc.residual(0, 0, 49)
    assert np.max(np.abs(r_dev - r_orc)) <= 1e-12 * np.max(np.abs(r_orc))


def test_scalar_kernel_known_answers():
    # test_kernels.cpp:39-47 and :86-96 with the ScalarLinear fixture
    hier = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, 5), [2], 2)
    drv = T.CycleDriver(T.ScalarLinear([0.5, 0.25], 1.0, False), hier, T.SolverConfig())
    drv.setup()
    drv.set_level(0, np.array([1, 9, 3, 9, 5.0]))
    drv.f_relax(0, 0, 2)
    assert drv.get_level(0)[:, 0].tolist() == [1, 0.5, 3, 1.5, 5]
    drv.set_level(0, np.array([1, 0.5, 3, 1.5, 5.0]))
    drv.c_relax(0, 0, 3)
    assert drv.get_level(0)[:, 0].tolist() == [1, 0.5, 0.25, 1.5, 0.75]
    drv.f_relax(0, 0, 2)
    assert drv.get_level(0)[:, 0].tolist() == [1, 0.5, 0.25, 0.125, 0.75]


def _golden_solve(name, workers=1, tol_hist=1e-9):
    case = golden_cases()[name]
    args = case["args"]
    ic = golden_array(name, "ic") if case.get("has_ic") else None
    files = {"w_file": golden_array(name, "w_file")} if args.get("functional") == "weights" else None
    app, hier, cfg = device_objects(args, ic=ic, files=files)
    res = T.solve(app, hier, cfg, workers=workers)
    assert res.report.converged == case["converged"]
    assert res.report.iterations == case["iterations"], (res.report.iterations, case["iterations"])
    hist = np.array(res.report.residual_norms)
    ref = np.array(case["history"])
    scale = ref[0]
    dev = np.abs(hist - ref) / np.maximum(np.abs(ref), 1e-300)
    ok = (dev <= tol_hist) | (np.abs(hist - ref) <= tol_hist * scale)
    assert ok.all(), (hist, ref)
    assert_final_state(name, case, res.state)
    return res


def assert_final_state(name, case, state):
    """Final-state bar against the compiled reference: the whole state when
    the fixture holds it, else every `row_stride`-th point row (plus the last)
    and the whole state's 2-norm, each within 1e-10 relative."""
    state = np.asarray(state).reshape(state.shape[0], -1)
    if case.get("store_u"):
        assert rel_l2(state, golden_array(name, "u")) <= SOLVE_RTOL
    stride = case.get("row_stride")
    if stride:
        idx = sorted(set(range(0, state.shape[0], stride)) | {state.shape[0] - 1})
        rows = golden_array(name, "rows")
        assert rows.shape == (len(idx), state.shape[1]), rows.shape
        # (not row by row: at t_f = 1 the heat solution has decayed ~1e-10-fold,
        # and both fp64 paths carry ~1e-18 absolute rounding from 2^14 steps)
        assert rel_l2(state[idx], rows) <= SOLVE_RTOL, rel_l2(state[idx], rows)
    if "u_l2" in case:
        l2 = float(np.linalg.norm(state))
        assert abs(l2 - case["u_l2"]) <= SOLVE_RTOL * case["u_l2"], (l2, case["u_l2"])


@pytest.mark.parametrize("name", ["functional_norm2", "functional_weights", "functional_norm2_5r"])
@pytest.mark.parametrize("workers", [1, 3])
def test_functional_change_matches_reference(name, workers):
    # NormKind::FunctionalChange (solver.cpp:380-396) with the reference CLI's
    # u.norm2() and a linear w.u: same iteration count as the compiled
    # reference; the stopping values are relative changes of nearly equal
    # numbers (cancellation amplifies the summation-order rounding of f), so
    # the history is held to 1e-6 relative
    _golden_solve(name, workers=workers, tol_hist=1e-6)


def test_config1_matches_reference():
    _golden_solve("config1")


def test_dahlquist_matches_reference():
    _golden_solve("dahlquist_cfg")


def test_heat_explicit_forcing_matches_reference():
    _golden_solve("heat_det_65")


def test_heat_full_single_matches_reference():
    _golden_solve("heat_full_single")


def test_fas_nested_fcf_matches_reference():
    _golden_solve("heat_fas_nested_fcf")


def test_fas_vcycle_substeps_matches_reference():
    _golden_solve("heat_fas_vcycle_f")


@pytest.mark.parametrize("name", ["heat_det_65", "heat_fas_nested_fcf", "config1"])
def test_histories_bitwise_across_shard_counts(name):
    # test_runtime.cpp:194-260: bit-identical histories and final state for any P
    case = golden_cases()[name]
    args = case["args"]
    ic = golden_array(name, "ic") if case.get("has_ic") else None
    base = None
    for workers in (1, 2, 4, 8):
        app, hier, cfg = device_objects(args, ic=ic)
        if workers > hier.n_coarsest_points():
            continue
        res = T.solve(app, hier, cfg, workers=workers)
        if base is None:
            base = res
            continue
        assert res.report.residual_norms == base.report.residual_norms, workers
        assert np.array_equal(res.state, base.state), workers


def test_fused_norm_equals_full_residual_norm():
    # the stopping norm sums the per-C-point squares the correction sweep's
    # tail wrote; the full residual norm re-evaluates every point (F residuals
    # are exactly zero after a cycle): the same squares, summed over arrays of
    # different length, hence a different fixed association -- equal to
    # rounding
    case = golden_cases()["heat_det_65"]
    app, hier, cfg = device_objects(case["args"])
    drv = T.CycleDriver(app, hier, cfg)
    drv.setup()
    norms = drv.iterate(3)
    full = drv.residual_norm()
    assert abs(full - norms[-1]) <= 4e-16 * full


def test_exact_in_nt_iterations_every_k():
    # test_solver.cpp:81-103
    grid = T.TimeGrid.make(0.0, 4.0, 65)
    for k in range(2, 10):
        hier = T.build_hierarchy(grid, [8], k)
        app = T.Dahlquist(-1.0, 1.0, False)
        cfg = T.SolverConfig(initial_guess=T.InitialGuess.Random, seed=99, tol=1e-300, max_iters=8)
        drv = T.CycleDriver(app, hier, cfg)
        drv.setup()
        for _ in range(8):
            drv.cycle()
        u = drv.get_level(0)[:, 0]
        mult = 1.0 / (1.0 + 4.0 / 64)
        exact = np.array([mult ** i for i in range(65)])
        assert np.max(np.abs(u - exact)) < 1e-12, k


def test_divergence_reports_iteration():
    hier = T.build_hierarchy(T.TimeGrid.make(0.0, 32.0, 33), [4], 3)
    cfg = T.SolverConfig(initial_guess=T.InitialGuess.Random, tol=1e-7)
    with pytest.raises(T.DivergenceError) as ei:
        T.solve(T.Dahlquist(1.0, 1.0, False), hier, cfg)
    assert ei.value.iteration == 1


def test_config5_shape_reduced_single_iteration():
    # n = 4095 with the BASELINE config-5 discretisation at N_t = 2^12: one
    # cycle on the device against the oracle's cycle (same inputs)
    n, npts = 4095, 4097
    ic = O.random_state(7, n)
    args = dict(problem="heat1d", n=n, tf=1.0, n_points=npts, m=16, k=8, manufactured=0,
                guess="random", seed=20, tol=1e-10, max_iters=2)
    app, hier, cfg = device_objects(args, ic=ic)
    drv = T.CycleDriver(app, hier, cfg)
    drv.setup()
    got = drv.iterate(2)
    orc = oracle_driver(args, ic=ic)
    orc.setup()
    want = []
    for _ in range(2):
        orc.cycle()
        want.append(orc.residual_norm())
    assert np.allclose(got, want, rtol=1e-9, atol=0)
    assert rel_l2(drv.get_level(0), orc.array(0)) <= SOLVE_RTOL


@pytest.mark.parametrize("k", [2, 4, 8, 12, 64, 128])
def test_heat_k_study_iteration_counts(k):
    # acceptance.cpp:158-201 (criterion 3), counts 45/24/14/14/14/14
    _golden_solve(f"kstudy_k{k}")


@pytest.mark.parametrize("m,k", [(16, 1), (16, 2), (16, 4), (16, 8), (16, 1025),
                                 (64, 1), (64, 2), (64, 4), (64, 8), (64, 257)])
def test_config5_shape_matches_reference(m, k):
    # BASELINE config 5 discretisation (n=4095) at N_t = 2^14, tol 1e-10, every
    # (m, k) cell incl. classical k = N_T + 1: same iteration count as the
    # compiled reference, history within 1e-9, final state (every 256th row,
    # the last row, the 2-norm) within 1e-10 relative l2
    _golden_solve(f"config5r_k{k}" if m == 16 else f"config5r_m{m}_k{k}")


def test_config5_shape_bitwise_across_shard_counts():
    case = golden_cases()["config5r_k8"]
    ic = golden_array("config5r_k8", "ic")
    args = dict(case["args"], max_iters=6, tol=1e-300)
    base = None
    for workers in (1, 2, 4, 8):
        app, hier, cfg = device_objects(args, ic=ic)
        drv = T.CycleDriver(app, hier, cfg, workers=workers)
        drv.setup()
        norms = drv.iterate(6)
        u = drv.get_level(0, first=16000, count=385)
        if base is None:
            base = (norms, u)
            continue
        assert np.array_equal(norms, base[0]), workers
        assert np.array_equal(u, base[1]), workers


def test_config5_shape_l32_windows_and_store_policies_against_the_reference(monkeypatch):
    # the config-5 shape (N_t = 2^14, k = 8) against the compiled reference's
    # fixture with the coarsest level on the L = 32 window kernel (two stream
    # buffers, emit by TMA reduce-add into the fine C row), and the level-0 row
    # stores under every L2 policy (the policy cannot change a value: bitwise)
    monkeypatch.setenv("ATM_WIN_L32", "1")
    a = _golden_solve("config5r_k8")
    monkeypatch.delenv("ATM_WIN_L32")
    states = []
    for hint in ("0", "1", "2"):
        monkeypatch.setenv("ATM_ST_HINT", hint)
        r = _golden_solve("config5r_k8")
        states.append((np.array(r.report.residual_norms), np.asarray(r.state)))
    for h, st in states[1:]:
        assert np.array_equal(h, states[0][0]) and np.array_equal(st, states[0][1])
    assert a.report.iterations == r.report.iterations


@pytest.mark.parametrize("n", [2047, 2048, 2049, 2053, 2056, 3001, 4090, 4095, 4096])
def test_two_level_solve_across_chunk_lengths(n):
    # n around the L = 16 / L = 32 switch (pitch > 2048) and the exact fit;
    # past 2048 the coarsest level's windows run the sub-block solve
    # (tri_solve_sb, two 8-element chains per chunk): n % 16 = 1, 5 puts the
    # row end inside the first sub-block of its thread (kappa of both
    # sub-blocks), 8 on the sub-block boundary, 9, 10, 15 inside the second
    # (dt/h^2 ~ 1000, the stiffness of the BASELINE configs; at 1e4 the
    # reference's own fp64 Thomas error alone reaches ~1e-10 of the state)
    args = dict(problem="heat1d", n=n, tf=1.0 / 64, n_points=257, m=8, k=4, manufactured=1,
                guess="random", seed=13, max_iters=60, tol=1e-9)
    app, hier, cfg = device_objects(args)
    res = T.solve(app, hier, cfg)
    orc = oracle_driver(args)
    ref = orc.drive()
    assert res.report.iterations == ref["iterations"]
    assert rel_l2(res.state, orc.array(0)) <= SOLVE_RTOL


@pytest.mark.parametrize("n", [4097, 5000, 5376, 5377, 8192, 12289, 32768, 65536])
def test_two_level_and_fas_solves_past_4096_unknowns(n):
    # 4096 < n <= 5376: rows padded to a multiple of 256 and moved as two
    # half-row TMA boxes; sweeps run L = 32 with 256 threads, the coarsest
    # level's windows L = 16 with up to 512.  n > 5376: rows split over a
    # cluster of ceil(n / 4096) CTAs coupled by a block Woodbury correction
    # (heat_cluster_host).  dt/h^2 ~ 1000, as the other final-state parity
    # cases
    tf = 1000.0 * 256 / (n + 1) ** 2
    for args in (dict(problem="heat1d", n=n, tf=tf, n_points=257, m=8, k=4, manufactured=1,
                      guess="random", seed=13, max_iters=60, tol=1e-9),
                 dict(problem="heat1d", n=n, folded=1, tf=tf, n_points=257, m="4,4", k=3, mode="v-cycle",
                      manufactured=1, guess="random", seed=17, max_iters=40, tol=1e-9)):
        app, hier, cfg = device_objects(args)
        res = T.solve(app, hier, cfg)
        orc = oracle_driver(args)
        ref = orc.drive()
        assert res.report.iterations == ref["iterations"], (args, res.report.iterations, ref["iterations"])
        assert rel_l2(res.state, orc.array(0)) <= SOLVE_RTOL


def test_fas_vcycle_mixed_chunk_lengths_matches_oracle():
    # n = 4095: levels 0-1 run L = 32 sweeps, the coarsest level L = 16
    # windows; level-l sweeps store restriction tails into level l+1 arrays
    args = dict(problem="heat1d", n=4095, folded=1, tf=1.0 / 32, n_points=513, m="4,4", k=3,
                mode="v-cycle", manufactured=1, guess="random", seed=17, max_iters=40, tol=1e-9)
    app, hier, cfg = device_objects(args)
    res = T.solve(app, hier, cfg)
    orc = oracle_driver(args)
    ref = orc.drive()
    assert res.report.iterations == ref["iterations"]
    assert rel_l2(res.state, orc.array(0)) <= SOLVE_RTOL


def test_cuda_graph_replay_bitwise_equals_direct_launches(monkeypatch):
    # cycles replayed from the captured CUDA graph produce bitwise the
    # directly launched cycles' histories and states
    args = dict(problem="heat1d", n=255, tf=1.0, n_points=1025, m=16, k=4, manufactured=1,
                guess="random", seed=3, max_iters=30, tol=1e-12)
    app, hier, cfg = device_objects(args)
    a = T.solve(app, hier, cfg)
    monkeypatch.setenv("ATM_NO_GRAPH", "1")
    b = T.solve(app, hier, cfg)
    assert a.report.iterations == b.report.iterations
    assert np.array_equal(np.array(a.report.residual_norms), np.array(b.report.residual_norms))
    assert np.array_equal(a.state, b.state)


@pytest.mark.parametrize("workers", [1, 3])
def test_relax_reuse_bitwise_equals_full_cycles(workers):
    # opt-in reuse of the correction sweep's C-point residuals as the next
    # cycle's restriction input: bitwise the same histories and states
    args = dict(problem="heat1d", n=1025, tf=1.0, n_points=2049, m=16, k=4, manufactured=1,
                guess="random", seed=21, max_iters=80, tol=1e-10)
    app, hier, cfg = device_objects(args)
    a = T.solve(app, hier, cfg, workers=workers)
    b = T.solve(app, hier, cfg, workers=workers, reuse_relax=True)
    assert a.report.iterations == b.report.iterations
    assert np.array_equal(np.array(a.report.residual_norms), np.array(b.report.residual_norms))
    assert np.array_equal(a.state, b.state)
    # reused cycles count one F-sweep of Phi applications, not two
    assert b.report.dof_steps < a.report.dof_steps


def test_relax_reuse_invalidated_by_set_level():
    args = dict(problem="heat1d", n=63, tf=1.0, n_points=257, m=8, k=3, manufactured=0,
                guess="random", seed=4, max_iters=20, tol=1e-14)
    app, hier, cfg = device_objects(args)
    drv_a = T.CycleDriver(app, hier, cfg)
    drv_b = T.CycleDriver(app, hier, cfg, reuse_relax=True)
    for d in (drv_a, drv_b):
        d.setup()
        d.iterate(2)
        u = d.get_level(0)
        u[5:40] *= 0.5  # perturb F and C points between cycles
        d.set_level(0, u)
    na, nb = drv_a.iterate(3), drv_b.iterate(3)
    assert np.array_equal(na, nb)
    assert np.array_equal(drv_a.get_level(0), drv_b.get_level(0))


@pytest.mark.parametrize("m,k", [(16, 8), (64, 4)])
def test_config5_shape_large_front_bound_and_sequential_state(m, k):
    """Config-5 shape at N_t = 2^16 (beyond what the CPU oracle finishes in
    seconds), size-independent properties: with a random guess the solve
    converges once the exact-C-point front has crossed the grid, i.e. in
    N_T/k (+1) iterations (test_solver.cpp:428-465), and the converged state
    equals sequential time stepping (a single interval, m = N_t, whose one
    F-relaxation IS u_i = Phi(u_{i-1})) to what the 1e-10 residual allows."""
    n, npts = 4095, 2 ** 16 + 1
    app = T.Heat1D(n, manufactured_forcing=False, initial_condition=T.random_state(7, n))
    rows = [npts // 4, npts // 2, npts - 1]
    seq_h = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, npts), [npts - 1], 2)
    seq = T.CycleDriver(app, seq_h, T.SolverConfig(relaxation=T.Relaxation.F, tol=1e-300, max_iters=1,
                                                   initial_guess=T.InitialGuess.Random, seed=20))
    seq.setup()
    seq.iterate(1)
    ref = {p: seq.get_level(0, first=p, count=1)[0] for p in rows}
    seq.close()
    n_t = (npts - 1) // m
    hier = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, npts), [m], k)
    cfg = T.SolverConfig(relaxation=T.Relaxation.F, tol=1e-10, max_iters=2 * n_t // k + 50,
                         initial_guess=T.InitialGuess.Random, seed=20)
    drv = T.CycleDriver(app, hier, cfg, reuse_relax=True, cpoint_storage=True)
    drv.setup()
    rep = drv.drive()
    assert rep.converged
    assert n_t // k <= rep.iterations <= n_t // k + 2, rep.iterations
    u0 = np.linalg.norm(T.random_state(7, n))
    for p in rows:
        err = np.linalg.norm(drv.get_level(0, first=p, count=1)[0] - ref[p]) / u0
        assert err < 1e-11, (p, err)
    drv.close()


@pytest.mark.parametrize("variant", ["fcf", "nested_fcf_substeps", "global_coarse", "shards",
                                     "reuse_cpoints"])
def test_cluster_rows_across_cycle_variants(variant):
    # rows split over a 2-CTA cluster (n = 6001) through every sweep / window
    # job kind: FCF (C-relaxation, stored C rows), nested FCF with coarse
    # sub-steps (forward windows, FAS right-hand sides), the global coarse
    # chain (k >= N_T + 1), three time shards, relax reuse + C-point storage
    n = 6001
    tf = 1000.0 * 64 / (n + 1) ** 2
    base = dict(problem="heat1d", n=n, tf=tf, n_points=129, m=8, k=4, manufactured=1,
                guess="random", seed=11, max_iters=60, tol=1e-9)
    kw = {}
    if variant == "fcf":
        args = dict(base, relax="FCF")
    elif variant == "nested_fcf_substeps":
        args = dict(base, folded=1, mode="nested-v", relax="FCF", m="4,4", k=3, substeps=2)
    elif variant == "global_coarse":
        args = dict(base, folded=1, mode="nested-v", m="8", k=40)
    elif variant == "shards":
        args = dict(base, mode="v-cycle", folded=1, m="4,4", k=3)
        kw = dict(workers=3)
    else:
        args = dict(base, manufactured=0)
        kw = dict(reuse_relax=True, cpoint_storage=True)
    app, hier, cfg = device_objects(args)
    res = T.solve(app, hier, cfg, **kw)
    orc = oracle_driver(args)
    ref = orc.drive()
    assert res.report.iterations == ref["iterations"], (variant, res.report.iterations, ref["iterations"])
    assert rel_l2(res.state, orc.array(0)) <= SOLVE_RTOL
