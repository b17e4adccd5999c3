"""`tempo_b200`, the flat-config front end (reference CLI: src/run_config.cpp:
295-413, include/tempo/cli.hpp:12-64) driving the GPU path through the C ABI.
Config errors are host-only (exit code 2); solves run on the GPU and are
checked against the compiled reference's golden iteration counts."""
from __future__ import annotations

import os
import subprocess

import numpy as np
import pytest

from conftest import golden_cases

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2107_09596_b200", "tempo_b200")


def run(tmp_path, text, cmd="solve", *extra):
    cfg = tmp_path / "run.cfg"
    cfg.write_text(text)
    p = subprocess.run([CLI, cmd, str(cfg), *extra], capture_output=True, text=True, timeout=600)
    return p.returncode, p.stdout, p.stderr


@pytest.mark.parametrize("text,needle", [
    ("problem = heat1d\nbogus.key = 1\n", "unknown key 'bogus.key'"),
    ("problem = heat1d\nproblem = heat1d\n", "duplicate key 'problem'"),
    ("problem = heat1d\nthis line has no equals\n", "expected 'key = value'"),
    ("problem = heat1d\nsolver.m = 4\nsolver.k = 2\ngrid.n_points = 33\nsolver.tol = 1e-9\n",
     "missing key 'grid.tf'"),
    ("problem = heat1d\nsolver.m = 4\nsolver.k = 2\ngrid.n_points = 33\nsolver.tol = 1e-9\n"
     "grid.tf = x\n", "is not a number"),
    ("problem = heat1d\nsolver.m = 4, y\nsolver.k = 2\n", "non-integer entry 'y'"),
    ("problem = heat1d\nsolver.m = 4\nsolver.k = 2\ngrid.n_points = 33\nsolver.tol = 1e-9\n"
     "grid.tf = 1\nsolver.mode = w-cycle\n", "solver.mode must be"),
    ("problem = lorenz\n", "unknown problem 'lorenz'"),
    ("problem = grayscott\ngrayscott.bogus = 1\n", "unknown key 'grayscott.bogus'"),
])
def test_cli_config_errors_exit_2(tmp_path, text, needle):
    code, _, err = run(tmp_path, text)
    assert code == 2, (code, err)
    assert needle in err


def test_cli_usage_exit_2():
    p = subprocess.run([CLI], capture_output=True, text=True)
    assert p.returncode == 2


def _rows(out):
    lines = out.strip().splitlines()
    assert lines[0] == "iter,residual_norm,seconds"
    i = lines.index("converged,iterations,total_seconds")
    hist = [float(l.split(",")[1]) for l in lines[1:i]]
    conv, iters, _ = lines[i + 1].split(",")
    return hist, int(conv), int(iters)


@pytest.mark.gpu
def test_cli_solve_dahlquist_matches_reference(tmp_path):
    # the reference's configs/dahlquist.cfg run (golden case dahlquist_cfg)
    case = golden_cases()["dahlquist_cfg"]
    code, out, err = run(tmp_path, "problem = dahlquist\ndahlquist.lambda = -1.0\ngrid.tf = 2.0\n"
                         "grid.n_points = 33\nsolver.mode = two-level\nsolver.m = 4\nsolver.k = 3\n"
                         "solver.tol = 1e-9\nsolver.initial_guess = random\nsolver.seed = 11\n"
                         "solver.max_iters = 40\n")
    assert code == 0, err
    hist, conv, iters = _rows(out)
    assert conv == 1 and iters == case["iterations"]
    np.testing.assert_allclose(hist, case["history"], rtol=1e-9)


@pytest.mark.gpu
def test_cli_solve_heat_full_single_matches_reference(tmp_path):
    case = golden_cases()["heat_full_single"]
    code, out, err = run(tmp_path, "problem = heat1d\nheat1d.dof = 1025\ngrid.tf = 3.0\n"
                         "grid.n_points = 16384\nsolver.mode = two-level\nsolver.m = 128\n"
                         "solver.k = 12\nsolver.tol = 1e-7\nsolver.initial_guess = random\n"
                         "solver.seed = 20\nsolver.max_iters = 200\n", "solve", "--workers", "2")
    assert code == 0, err
    hist, conv, iters = _rows(out)
    assert iters == case["iterations"]
    ref = np.array(case["history"])
    # relative 1e-9, or 1e-9 of the first norm (the late norms sit near the
    # rounding floor of the sweep)
    assert np.all(np.abs(np.array(hist) - ref) <= 1e-9 * np.maximum(np.abs(ref), ref[0]))


@pytest.mark.gpu
def test_cli_sweep_k_matches_reference_k_study(tmp_path):
    # the k-study of configs/heat_k_study.cfg (k = 2, 4, 8, 12, 64, 128)
    cases = golden_cases()
    want = {k: cases[f"kstudy_k{k}"]["iterations"] for k in (2, 4, 8, 12, 64, 128)}
    code, out, err = run(tmp_path, "problem = heat1d\nheat1d.dof = 1025\ngrid.tf = 3.0\n"
                         "grid.n_points = 16384\nsolver.mode = two-level\nsolver.tol = 1e-7\n"
                         "solver.initial_guess = random\nsolver.seed = 20\nsolver.max_iters = 300\n"
                         "sweep.m_values = 128\nsweep.k_values = 2, 4, 8, 12, 64, 0\n", "sweep-k")
    assert code == 0, err
    lines = out.strip().splitlines()
    assert lines[0] == "m,k,k_over_ncpoints,iterations,parareal_equivalent"
    got = {int(l.split(",")[1]): int(l.split(",")[3]) for l in lines[1:]}
    # k = 0 selects the full coarse grid: 128 coarse points
    assert got == {2: want[2], 4: want[4], 8: want[8], 12: want[12], 64: want[64], 128: want[128]}
    assert lines[-1].endswith(",1")


@pytest.mark.gpu
def test_cli_not_converged_exit_1(tmp_path):
    code, out, _ = run(tmp_path, "problem = heat1d\nheat1d.dof = 63\ngrid.tf = 1.0\n"
                       "grid.n_points = 1025\nsolver.m = 16\nsolver.k = 2\nsolver.tol = 1e-14\n"
                       "solver.initial_guess = random\nsolver.seed = 20\nsolver.max_iters = 3\n")
    assert code == 1
    _, conv, iters = _rows(out)
    assert conv == 0 and iters == 3


@pytest.mark.gpu
def test_cli_grayscott_desk_matches_oracle(tmp_path):
    # configs/grayscott_desk.cfg (the paper's desk-scale run); iteration
    # count from the oracle restatement (the reference needs Eigen)
    from oracle import oracle as O
    orc = O.Driver(dict(kind=O.GRAY_SCOTT, nx=32), dict(tf=64.0, n_points=512, m=[16], k=16),
                   dict(mode=O.NESTED_V, tol=1e-7, max_iters=60))
    want = orc.drive()
    code, out, err = run(tmp_path, "problem = grayscott\ngrayscott.n = 32\ngrid.tf = 64.0\n"
                         "grid.n_points = 512\nsolver.mode = nested-v\nsolver.m = 16\nsolver.k = 16\n"
                         "solver.tol = 1e-7\nsolver.max_iters = 60\nruntime.workers = 1\n")
    assert code == 0, err
    hist, conv, iters = _rows(out)
    assert conv == 1 and iters == want["iterations"]
    np.testing.assert_allclose(hist, want["history"], rtol=1e-6)


@pytest.mark.gpu
def test_cli_trace_rows(tmp_path):
    trace = tmp_path / "trace.csv"
    code, out, err = run(tmp_path, "problem = heat1d\nheat1d.dof = 63\ngrid.tf = 1.0\n"
                         "grid.n_points = 257\nsolver.m = 16\nsolver.k = 2\nsolver.tol = 1e-9\n"
                         "solver.initial_guess = random\nsolver.seed = 20\nsolver.max_iters = 50\n"
                         f"runtime.trace = {trace}\n")
    assert code == 0, err
    _, _, iters = _rows(out)
    rows = trace.read_text().strip().splitlines()
    assert rows[0] == "iter,rank,phase,seconds"
    phases = {}
    for r in rows[1:]:
        it, rank, ph, sec = r.split(",")
        assert 1 <= int(it) <= iters and rank == "0" and float(sec) > 0.0
        phases.setdefault(ph, set()).add(int(it))
    for ph in ("relax", "restrict", "coarse", "correct", "norm"):
        assert phases.get(ph) == set(range(1, iters + 1)), ph


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,iters", [("grayscott_paper_two_level.cfg", 9),
                                       ("grayscott_paper_three_level.cfg", 7)])
def test_cli_grayscott_paper_runs_reproduce_published_iteration_counts(tmp_path, cfg, iters):
    # PAPER.md tab:gray_two_level (m = 128, k = 64: 9 iterations) and
    # tab:gray_three_level ((64, 4), k = 32, FCF: 7 iterations), 128^2 grid,
    # 16 384 time points -- the paper's own experiment, from configs/
    text = open(os.path.join(ROOT, "configs", cfg)).read()
    code, out, err = run(tmp_path, text)
    assert code == 0, err
    hist, conv, n = _rows(out)
    assert conv == 1 and n == iters, (n, hist)
