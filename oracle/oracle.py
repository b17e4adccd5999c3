"""ctypes wrapper of the C oracle (atm_oracle.c) and the compiled reference
driver (_ref/tempo_ref).

TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, always as the checker or the
CPU baseline -- never by the product package paper_2107_09596_b200.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_BIN = os.path.join(HERE, "_ref", "tempo_ref")

HEAT1D, DAHLQUIST, SCALAR, ALLEN_CAHN, HEAT2D, GRAY_SCOTT = 1, 2, 3, 4, 5, 6
TWO_LEVEL, VCYCLE, NESTED_V = 0, 1, 2
RELAX_F, RELAX_FCF = 0, 1
NORM_L2, NORM_FUNCTIONAL = 0, 1
GUESS_CONSTANT, GUESS_RANDOM, GUESS_PROVIDED = 0, 1, 2
MAXL = 8

_DP = C.POINTER(C.c_double)


class Problem(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("n", C.c_int), ("folded", C.c_int),
        ("x0", C.c_double), ("x1", C.c_double), ("manufactured", C.c_int),
        ("lam", C.c_double), ("u0", C.c_double),
        ("n_mult", C.c_int), ("mult", C.c_double * MAXL),
        ("fine_forcing", _DP), ("n_ff", C.c_int),
        ("eps", C.c_double), ("length", C.c_double),
        ("newton_tol", C.c_double), ("newton_max", C.c_int),
        ("nx", C.c_int), ("cg_rtol", C.c_double), ("cg_max", C.c_int),
        ("source", _DP), ("ic", _DP),
        ("gs_domain", C.c_double), ("gs_feed", C.c_double), ("gs_kill", C.c_double),
        ("gs_du", C.c_double), ("gs_dv", C.c_double), ("gs_linear_tol", C.c_double),
        ("gs_reaction", C.c_int), ("gs_bounds_check", C.c_int),
        ("gs_bound_lo", C.c_double), ("gs_bound_hi", C.c_double),
    ]


class Grid(C.Structure):
    _fields_ = [("t0", C.c_double), ("tf", C.c_double), ("n_points", C.c_int),
                ("n_m", C.c_int), ("m", C.c_int * MAXL), ("k", C.c_int)]


class Solver(C.Structure):
    _fields_ = [("mode", C.c_int), ("relaxation", C.c_int), ("nu", C.c_int),
                ("max_iters", C.c_int), ("tol", C.c_double), ("norm", C.c_int),
                ("functional_w", _DP), ("initial_guess", C.c_int),
                ("seed", C.c_uint64), ("constant_value", _DP), ("provided", _DP),
                ("coarse_substeps", C.c_int)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            subprocess.check_call(["make", "-s", "-C", HERE, "oracle"])
        L = C.CDLL(LIB_PATH)
        L.orc_create.restype = C.c_void_p
        L.orc_create.argtypes = [C.POINTER(Problem), C.POINTER(Grid), C.POINTER(Solver),
                                 C.POINTER(C.c_int)]
        L.orc_create_error.restype = C.c_char_p
        L.orc_error.restype = C.c_char_p
        L.orc_error.argtypes = [C.c_void_p]
        L.orc_destroy.argtypes = [C.c_void_p]
        for f in ("orc_setup", "orc_cycle", "orc_nested_init"):
            getattr(L, f).argtypes = [C.c_void_p]
        L.orc_residual_norm.argtypes = [C.c_void_p, _DP]
        L.orc_drive.argtypes = [C.c_void_p, _DP, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.orc_array.restype = _DP
        L.orc_array.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.orc_n_levels.argtypes = [C.c_void_p]
        L.orc_vector_size.argtypes = [C.c_void_p]
        L.orc_step.argtypes = [C.c_void_p, C.c_int, C.c_int, _DP, _DP]
        L.orc_forcing.argtypes = [C.c_void_p, C.c_int, C.c_int, _DP]
        L.orc_initial_condition.argtypes = [C.c_void_p, _DP]
        L.orc_random_state.argtypes = [C.c_uint64, C.c_int, _DP]
        L.orc_level_points.argtypes = [C.POINTER(Grid), C.c_int]
        L.orc_k_f_relax.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int]
        L.orc_k_c_relax.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int]
        L.orc_k_residual.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, _DP]
        L.orc_k_window_linear.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, _DP, _DP]
        L.orc_k_window_fas.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, _DP, _DP, _DP]
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(_DP)


def random_state(seed: int, n: int) -> np.ndarray:
    """splitmix64 fill restated in atm_oracle.c (state_vector.hpp:108-118)."""
    out = np.empty(n, dtype=np.float64)
    lib().orc_random_state(C.c_uint64(seed), n, _ptr(out))
    return out


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class Driver:
    """Sequential CycleDriver restatement over one problem/grid/solver."""

    def __init__(self, problem: dict, grid: dict, solver: dict):
        self._keep = []
        p = Problem()
        p.kind = problem["kind"]
        p.n = problem.get("n", 1)
        p.folded = int(problem.get("folded", 0))
        p.x0, p.x1 = problem.get("x0", 0.0), problem.get("x1", 1.0)
        p.manufactured = int(problem.get("manufactured", 1))
        p.lam, p.u0 = problem.get("lam", -1.0), problem.get("u0", 1.0)
        mult = problem.get("mult", [])
        p.n_mult = len(mult)
        for i, v in enumerate(mult):
            p.mult[i] = v
        p.eps, p.length = problem.get("eps", 0.02), problem.get("length", 1.0)
        p.newton_tol, p.newton_max = problem.get("newton_tol", 1e-12), problem.get("newton_max", 30)
        p.nx, p.cg_rtol, p.cg_max = problem.get("nx", 0), problem.get("cg_rtol", 1e-12), problem.get("cg_max", 10000)
        # gray-scott (gray_scott.hpp:24-38 defaults)
        p.gs_domain, p.gs_feed = problem.get("domain", 2.5), problem.get("feed", 0.024)
        p.gs_kill, p.gs_du, p.gs_dv = problem.get("kill", 0.06), problem.get("du", 8e-5), problem.get("dv", 4e-5)
        p.gs_linear_tol = problem.get("linear_tol", 1e-10)
        p.gs_reaction, p.gs_bounds_check = int(problem.get("reaction", 1)), int(problem.get("bounds_check", 1))
        p.gs_bound_lo, p.gs_bound_hi = problem.get("bound_lo", -1.0), problem.get("bound_hi", 3.0)
        if problem["kind"] == GRAY_SCOTT and "newton_tol" not in problem:
            p.newton_tol = 1e-10
        for key, field, cnt in (("fine_forcing", "fine_forcing", "n_ff"), ("source", "source", None),
                                ("ic", "ic", None)):
            if problem.get(key) is not None:
                a = np.ascontiguousarray(problem[key], dtype=np.float64)
                self._keep.append(a)
                setattr(p, field, _ptr(a))
                if cnt:
                    setattr(p, cnt, a.size)
        g = Grid()
        g.t0, g.tf, g.n_points = grid.get("t0", 0.0), grid["tf"], grid["n_points"]
        ms = grid["m"] if isinstance(grid["m"], (list, tuple)) else [grid["m"]]
        g.n_m = len(ms)
        for i, v in enumerate(ms):
            g.m[i] = v
        g.k = grid["k"]
        s = Solver()
        s.mode = solver.get("mode", TWO_LEVEL)
        s.relaxation = solver.get("relaxation", RELAX_F)
        s.nu = solver.get("nu", 1)
        s.max_iters = solver.get("max_iters", 100)
        s.tol = solver.get("tol", 1e-7)
        s.norm = solver.get("norm", NORM_L2)
        s.initial_guess = solver.get("initial_guess", GUESS_CONSTANT)
        s.seed = solver.get("seed", 0)
        s.coarse_substeps = solver.get("coarse_substeps", 1)
        for key in ("functional_w", "constant_value", "provided"):
            if solver.get(key) is not None:
                a = np.ascontiguousarray(solver[key], dtype=np.float64)
                self._keep.append(a)
                setattr(s, key, _ptr(a))
        self.max_iters = s.max_iters
        st = C.c_int(0)
        self.h = lib().orc_create(C.byref(p), C.byref(g), C.byref(s), C.byref(st))
        if not self.h:
            raise OracleError(st.value, lib().orc_create_error().decode())
        self.grid = g
        self.L = lib().orc_n_levels(self.h)
        self.n = lib().orc_vector_size(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_destroy(self.h)
            self.h = None

    def _check(self, st):
        if st not in (0, 1):
            raise OracleError(st, lib().orc_error(self.h).decode())
        return st

    def points(self, level):
        return lib().orc_level_points(C.byref(self.grid), level)

    def setup(self):
        self._check(lib().orc_setup(self.h))

    def cycle(self):
        self._check(lib().orc_cycle(self.h))

    def nested_init(self):
        self._check(lib().orc_nested_init(self.h))

    def residual_norm(self):
        out = C.c_double()
        self._check(lib().orc_residual_norm(self.h, C.byref(out)))
        return out.value

    def drive(self):
        hist = np.zeros(self.max_iters, dtype=np.float64)
        it, conv = C.c_int(), C.c_int()
        st = lib().orc_drive(self.h, _ptr(hist), C.byref(it), C.byref(conv))
        if st not in (0, 1):
            err = OracleError(st, lib().orc_error(self.h).decode())
            # completed iterations and their norms before the failing cycle
            err.iterations, err.history = it.value, hist[: it.value].copy()
            raise err
        return dict(iterations=it.value, converged=bool(conv.value),
                    history=hist[: it.value].copy())

    def array(self, level, which="u"):
        w = {"u": 0, "g": 1, "v": 2, "r": 3}[which]
        ptr = lib().orc_array(self.h, level, w)
        if not ptr:
            raise ValueError("array not allocated (call setup first)")
        cnt = self.points(level) * self.n
        return np.ctypeslib.as_array(ptr, shape=(cnt,)).reshape(self.points(level), self.n)

    def step(self, level, index, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty_like(x)
        self._check(lib().orc_step(self.h, level, index, _ptr(x), _ptr(out)))
        return out

    def forcing(self, level, index):
        out = np.empty(self.n, dtype=np.float64)
        self._check(lib().orc_forcing(self.h, level, index, _ptr(out)))
        return out

    def initial_condition(self):
        out = np.empty(self.n, dtype=np.float64)
        lib().orc_initial_condition(self.h, _ptr(out))
        return out

    # kernels.cpp restatements on the driver's own arrays
    def f_relax(self, level, first, count):
        self._check(lib().orc_k_f_relax(self.h, level, first, count))

    def c_relax(self, level, first, count):
        self._check(lib().orc_k_c_relax(self.h, level, first, count))

    def residual(self, level, first, count):
        out = np.empty((count, self.n), dtype=np.float64)
        self._check(lib().orc_k_residual(self.h, level, first, count, _ptr(out)))
        return out

    def window_linear(self, level, lo, r_win):
        r_win = np.ascontiguousarray(r_win, dtype=np.float64)
        out = np.empty(self.n, dtype=np.float64)
        self._check(lib().orc_k_window_linear(self.h, level, lo, r_win.shape[0], _ptr(r_win), _ptr(out)))
        return out

    def window_fas(self, level, lo, v_win, r_win):
        v_win = np.ascontiguousarray(v_win, dtype=np.float64)
        r_win = np.ascontiguousarray(r_win, dtype=np.float64)
        out = np.empty(self.n, dtype=np.float64)
        self._check(lib().orc_k_window_fas(self.h, level, lo, v_win.shape[0], _ptr(v_win),
                                           _ptr(r_win), _ptr(out)))
        return out


# --------------------------------------------------------------------------
# compiled reference driver (_ref/tempo_ref)

def ref_available() -> bool:
    return os.path.exists(REF_BIN)


def run_ref(args: dict, out_u: bool = False, files: dict | None = None, timeout=3600):
    """Run the compiled reference with key=value args; returns (json, u or None)."""
    tmp = tempfile.mkdtemp(prefix="tempo_ref_")
    argv = [REF_BIN]
    for k, v in (files or {}).items():
        path = os.path.join(tmp, k + ".bin")
        np.ascontiguousarray(v, dtype=np.float64).tofile(path)
        argv.append(f"{k}={path}")
    upath = os.path.join(tmp, "u.bin")
    if out_u:
        argv.append(f"out_u={upath}")
    argv += [f"{k}={v}" for k, v in args.items()]
    proc = subprocess.run(argv, capture_output=True, text=True, timeout=timeout)
    line = proc.stdout.strip().splitlines()[-1] if proc.stdout.strip() else "{}"
    res = json.loads(line)
    u = np.fromfile(upath, dtype=np.float64) if out_u and os.path.exists(upath) else None
    return res, u
