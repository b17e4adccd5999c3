"""Reference-shaped host API over the C ABI (include/atmgrit.h).

Names, argument meaning and error behaviour follow the reference `tempo`
library (/root/reference/proj/include/tempo/*.hpp) so tests read like the
reference's own: TimeGrid.make, build_hierarchy, SolverConfig, CycleDriver
(setup / cycle / nested_init / residual_norm / drive), solve(),
run_parallel(), problems.Heat1D / Dahlquist, and the ScalarLinear fixture.
All arithmetic happens in libatmgrit.so on the GPU; this module only marshals.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
from typing import Optional, Sequence

import numpy as np

from . import _capi
from ._capi import lib, ptr

# ---------------------------------------------------------------------------
# errors (errors.hpp:9-42)


class TempoError(RuntimeError):
    pass


class ConfigError(TempoError):
    pass


class DivergenceError(TempoError):
    def __init__(self, iteration: int, what: str):
        super().__init__(what)
        self.iteration = iteration


class RuntimeFault(TempoError):
    pass


class NonlinearSolveError(TempoError):
    pass


def _raise(status: int, msg: str, iteration: int = 0):
    if status == 2:
        raise ConfigError(msg)
    if status == 4:
        import re
        m = re.search(r"iteration (\d+)", msg)
        raise DivergenceError(int(m.group(1)) if m else iteration, msg)
    if status == 5:
        raise NonlinearSolveError(msg)
    raise RuntimeFault(msg)


# ---------------------------------------------------------------------------
# grids (time_grid.hpp, hierarchy.hpp)


@dataclasses.dataclass
class TimeGrid:
    t0: float
    tf: float
    n_points: int
    dt: float

    @staticmethod
    def make(t0: float, tf: float, n_points: int) -> "TimeGrid":
        if n_points < 2:
            raise ConfigError("TimeGrid: need at least 2 points")
        if not tf > t0:
            raise ConfigError("TimeGrid: tf must exceed t0")
        return TimeGrid(t0, tf, n_points, (tf - t0) / float(n_points - 1))

    def n_steps(self):
        return self.n_points - 1


@dataclasses.dataclass
class CfSplit:
    m: int
    c_points: list
    intervals: list  # (c_left, first, last)


def make_cf_split(n_points: int, m: int) -> CfSplit:
    """hierarchy.cpp:7-22."""
    if m < 2:
        raise ConfigError(f"coarsening factor must exceed 1, got {m}")
    if n_points < 2:
        raise ConfigError("cannot split a level with fewer than 2 points")
    last = n_points - 1
    cps = list(range(0, last + 1, m))
    ivs = [(c, c + 1, min(c + m - 1, last)) for c in cps if c + 1 <= min(c + m - 1, last)]
    return CfSplit(m, cps, ivs)


@dataclasses.dataclass
class LocalCoarseGrid:
    owner: int
    lo: int

    def size(self):
        return self.owner - self.lo + 1


class Hierarchy:
    """build_hierarchy(fine, m, k) (hierarchy.cpp:24-50)."""

    def __init__(self, fine: TimeGrid, m: Sequence[int], k: int):
        if len(m) == 0:
            raise ConfigError("hierarchy needs at least one coarsening factor")
        if k < 1:
            raise ConfigError("local-grid distance k must be at least 1")
        self.fine = fine
        self.m = list(m)
        self._k = k
        self.levels = [fine]
        self.splits = []
        for l, ml in enumerate(self.m):
            cur = self.levels[-1]
            self.splits.append(make_cf_split(cur.n_points, ml))
            nc = (cur.n_points - 1) // ml + 1
            if nc < 2:
                raise ConfigError(f"coarsening exhausts the grid at level {l + 1} ({nc} points)")
            dt = cur.dt * ml
            self.levels.append(TimeGrid(cur.t0, cur.t0 + dt * (nc - 1), nc, dt))

    def n_levels(self):
        return len(self.levels)

    def level(self, l):
        return self.levels[l]

    def k(self):
        return self._k

    def split(self, l):
        return self.splits[l]

    def coarsest(self):
        return self.n_levels() - 1

    def n_coarsest_points(self):
        return self.levels[-1].n_points

    def local_grid(self, p):
        return LocalCoarseGrid(p, max(0, p - self._k + 1))

    def is_global_coarse_grid(self):
        return self._k >= self.n_coarsest_points()

    def coarsening_factors(self):
        return list(self.m)

    def c_grid(self) -> _capi.atm_grid:
        g = _capi.atm_grid()
        g.t0, g.tf, g.n_points = self.fine.t0, self.fine.tf, self.fine.n_points
        g.n_m = len(self.m)
        for i, v in enumerate(self.m):
            g.m[i] = v
        g.k = self._k
        return g


def build_hierarchy(fine: TimeGrid, m: Sequence[int], k: int) -> Hierarchy:
    return Hierarchy(fine, m, k)


# ---------------------------------------------------------------------------
# solver configuration (solver_config.hpp:14-68)


class CycleMode(enum.IntEnum):
    TwoLevel = 0
    VCycle = 1
    NestedV = 2


class Relaxation(enum.IntEnum):
    F = 0
    FCF = 1


class NormKind(enum.IntEnum):
    ResidualL2 = 0
    FunctionalChange = 1


class InitialGuess(enum.IntEnum):
    Constant = 0
    Random = 1
    Provided = 2


class StopReason(enum.IntEnum):
    Converged = 0
    MaxIterations = 1
    Diverged = 2


@dataclasses.dataclass
class SolverConfig:
    mode: CycleMode = CycleMode.TwoLevel
    relaxation: Relaxation = Relaxation.F
    nu: int = 1
    max_iters: int = 100
    tol: float = 1e-7
    norm: NormKind = NormKind.ResidualL2
    # FunctionalChange functional f(u): weights w of a linear functional w . u,
    # or the string "norm2" for u.norm2() (the reference CLI's, run_config.cpp:241-243)
    functional: Optional[object] = None
    initial_guess: InitialGuess = InitialGuess.Constant
    seed: int = 0
    constant_value: Optional[np.ndarray] = None
    provided: Optional[np.ndarray] = None  # [n_points, n]
    coarse_substeps: int = 1


@dataclasses.dataclass
class ConvergenceReport:
    residual_norms: list
    iterations: int = 0
    converged: bool = False
    stop_reason: StopReason = StopReason.MaxIterations
    total_seconds: float = 0.0
    dof_steps: float = 0.0
    timings: dict = dataclasses.field(default_factory=dict)
    iteration_seconds: list = dataclasses.field(default_factory=list)


# ---------------------------------------------------------------------------
# problems (the device Phi descriptor of an Application)


class Application:
    kind = 0

    def vector_size(self) -> int:
        raise NotImplementedError

    def forcing_folded(self) -> bool:
        raise NotImplementedError

    def c_problem(self, keep: list) -> _capi.atm_problem:
        raise NotImplementedError


class Heat1D(Application):
    """problems::Heat1D (heat1d.hpp:20-76) with an optional IC override."""
    kind = 1

    def __init__(self, n_dof=1025, x0=0.0, x1=1.0, folded=False, manufactured_forcing=True,
                 initial_condition=None):
        if n_dof < 1:
            raise ConfigError("heat1d: need at least one spatial unknown")
        if not x1 > x0:
            raise ConfigError("heat1d: x1 must exceed x0")
        self.n_dof, self.x0, self.x1 = n_dof, x0, x1
        self.folded = folded
        self.manufactured_forcing = manufactured_forcing
        self.ic = None if initial_condition is None else np.ascontiguousarray(initial_condition, np.float64)

    def vector_size(self):
        return self.n_dof

    def forcing_folded(self):
        return self.folded

    def mesh_width(self):
        return (self.x1 - self.x0) / (self.n_dof + 1)

    def c_problem(self, keep):
        p = _capi.atm_problem()
        p.kind, p.n, p.folded = self.kind, self.n_dof, int(self.folded)
        p.x0, p.x1, p.manufactured = self.x0, self.x1, int(self.manufactured_forcing)
        if self.ic is not None:
            keep.append(self.ic)
            p.ic = ptr(self.ic)
        return p


class Dahlquist(Application):
    """problems::Dahlquist (dahlquist.hpp:12-50)."""
    kind = 2

    def __init__(self, lam=-1.0, u0=1.0, folded=False):
        self.lam, self.u0, self.folded = lam, u0, folded

    def vector_size(self):
        return 1

    def forcing_folded(self):
        return self.folded

    def c_problem(self, keep):
        p = _capi.atm_problem()
        p.kind, p.n, p.folded, p.lam, p.u0 = self.kind, 1, int(self.folded), self.lam, self.u0
        return p


class ScalarLinear(Application):
    """The reference's scalar test fixture (tests/support.hpp:19-60)."""
    kind = 3

    def __init__(self, multipliers, u0=1.0, folded=False, fine_forcing=None):
        self.mult = list(multipliers)
        self.u0, self.folded = u0, folded
        self.ff = None if fine_forcing is None else np.ascontiguousarray(fine_forcing, np.float64)

    def vector_size(self):
        return 1

    def forcing_folded(self):
        return self.folded

    def c_problem(self, keep):
        p = _capi.atm_problem()
        p.kind, p.n, p.folded, p.u0 = self.kind, 1, int(self.folded), self.u0
        p.n_mult = len(self.mult)
        for i, v in enumerate(self.mult):
            p.mult[i] = v
        if self.ff is not None and self.ff.size:
            keep.append(self.ff)
            p.fine_forcing, p.n_ff = ptr(self.ff), self.ff.size
        return p


class AllenCahn(Application):
    """1D Allen-Cahn u_t = eps^2 u_xx + u - u^3, periodic on [0, length)
    (BASELINE config 3; no reference Phi, see oracle/atm_oracle.c ac_step).
    Backward Euler per sub-step, Newton with the stopping rule of
    gray_scott.cpp:113 (stop = max(tol, tol |F_0|)) and its iteration cap
    (NonlinearSolveError, gray_scott.cpp:165-169).  Forcing is folded (zero)."""
    kind = 4

    def __init__(self, n=4096, eps=0.02, length=1.0, newton_tol=1e-12, newton_max=30,
                 initial_condition=None):
        if n < 16 or n > 4096:
            raise ConfigError("allen-cahn: n must be in [16, 4096]")
        if not (eps > 0.0 and length > 0.0):
            raise ConfigError("allen-cahn: bad eps/length")
        self.n, self.eps, self.length = n, eps, length
        self.newton_tol, self.newton_max = newton_tol, newton_max
        self.ic = None if initial_condition is None else np.ascontiguousarray(initial_condition, np.float64)

    def vector_size(self):
        return self.n

    def forcing_folded(self):
        return True

    def c_problem(self, keep):
        p = _capi.atm_problem()
        p.kind, p.n, p.folded = self.kind, self.n, 1
        p.eps, p.length = self.eps, self.length
        p.newton_tol, p.newton_max = self.newton_tol, self.newton_max
        if self.ic is not None:
            keep.append(self.ic)
            p.ic = ptr(self.ic)
        return p


class GrayScott(Application):
    """problems::GrayScott (gray_scott.hpp:12-68): 2D Gray-Scott reaction-
    diffusion on [0, domain]^2, periodic, n x n cells, state [u; v], backward
    Euler with Newton (stop = max(tol, tol |F_0|), cap) and Jacobi-
    preconditioned BiCGSTAB inner solves; the bounds check of step().
    Forcing is folded.  The reference delegates BiCGSTAB to Eigen (absent
    here); the oracle restates the published algorithm (parity unpinned)."""
    kind = 6

    def __init__(self, n=32, domain=2.5, feed=0.024, kill=0.06, du=8e-5, dv=4e-5, newton_tol=1e-10,
                 newton_max_iters=30, linear_tol=1e-10, reaction=True, bounds_check=True,
                 bound_lo=-1.0, bound_hi=3.0, initial_condition=None):
        if n < 4:
            raise ConfigError("gray-scott: grid must be at least 4x4")
        if not domain > 0.0:
            raise ConfigError("gray-scott: domain size must be positive")
        self.n, self.domain, self.feed, self.kill, self.du, self.dv = n, domain, feed, kill, du, dv
        self.newton_tol, self.newton_max_iters, self.linear_tol = newton_tol, newton_max_iters, linear_tol
        self.reaction, self.bounds_check = reaction, bounds_check
        self.bound_lo, self.bound_hi = bound_lo, bound_hi
        self.ic = None if initial_condition is None else np.ascontiguousarray(initial_condition, np.float64).ravel()

    def vector_size(self):
        return 2 * self.n * self.n

    def forcing_folded(self):
        return True

    def c_problem(self, keep):
        p = _capi.atm_problem()
        p.kind, p.n, p.folded, p.nx = self.kind, 2 * self.n * self.n, 1, self.n
        p.newton_tol, p.newton_max = self.newton_tol, self.newton_max_iters
        p.gs_domain, p.gs_feed, p.gs_kill = self.domain, self.feed, self.kill
        p.gs_du, p.gs_dv, p.gs_linear_tol = self.du, self.dv, self.linear_tol
        p.gs_reaction, p.gs_bounds_check = int(self.reaction), int(self.bounds_check)
        p.gs_bound_lo, p.gs_bound_hi = self.bound_lo, self.bound_hi
        if self.ic is not None:
            keep.append(self.ic)
            p.ic = ptr(self.ic)
        return p


class Heat2D(Application):
    """2D heat u_t = Lap(u) + f on the unit square, nx x nx interior points,
    5-point stencil, zero Dirichlet (BASELINE configs 2 and 4; no reference
    Phi, see oracle/atm_oracle.c h2_solve).  Backward Euler per sub-step
    solved by matrix-free CG to |r| <= cg_rtol |b| from x0 = u_prev; the
    source enters as forcing(level, i) = A^{-1}(dt f) (explicit) or inside
    Phi (folded), like heat1d.cpp:66-100."""
    kind = 5

    def __init__(self, nx=127, folded=False, source=None, cg_rtol=1e-12, cg_max=10000,
                 initial_condition=None):
        if nx < 1:
            raise ConfigError("heat2d: need at least one interior point per side")
        self.nx, self.folded = nx, folded
        self.cg_rtol, self.cg_max = cg_rtol, cg_max
        self.source = None if source is None else np.ascontiguousarray(source, np.float64).ravel()
        self.ic = None if initial_condition is None else np.ascontiguousarray(initial_condition, np.float64).ravel()

    def vector_size(self):
        return self.nx * self.nx

    def forcing_folded(self):
        return self.folded

    def c_problem(self, keep):
        p = _capi.atm_problem()
        p.kind, p.n, p.folded = self.kind, self.nx * self.nx, int(self.folded)
        p.nx, p.cg_rtol, p.cg_max = self.nx, self.cg_rtol, self.cg_max
        for arr, field in ((self.source, "source"), (self.ic, "ic")):
            if arr is not None:
                keep.append(arr)
                setattr(p, field, ptr(arr))
        return p


# ---------------------------------------------------------------------------
# the driver


class _LevelView:
    """Lazy per-level array view pulled from the device (space_time.hpp:20-32)."""

    def __init__(self, drv, level):
        self._d, self._l = drv, level

    def _get(self, which):
        return self._d.get_level(self._l, which)

    @property
    def u(self):
        return self._get(0)

    @property
    def g(self):
        return self._get(1)

    @property
    def v(self):
        return self._get(2)

    @property
    def r(self):
        return self._get(3)


class _StateView:
    def __init__(self, drv):
        self._d = drv

    def level(self, l):
        return _LevelView(self._d, l)


class CycleDriver:
    """CycleDriver (solver.hpp:67-120) backed by the device engine.

    `workers` > 1 drives that many time shards (the reference's rank layout,
    layout.cpp:29-63) with device-to-device exchanges; `world_size` > 1 runs
    one shard per process with NCCL between processes.
    """

    def __init__(self, app: Application, hier: Hierarchy, cfg: SolverConfig, workers: int = 1,
                 device: int = 0, trace: bool = False, world_size: int = 1, rank: int = 0,
                 nccl_id: Optional[bytes] = None, reuse_relax: bool = False,
                 cpoint_storage: bool = False, defer_guess: bool = False, timeout_ms: int = 0):
        self.app, self.hier, self.cfg = app, hier, cfg
        self._keep = []
        p = app.c_problem(self._keep)
        g = hier.c_grid()
        s = _capi.atm_solver()
        s.mode, s.relaxation, s.nu = int(cfg.mode), int(cfg.relaxation), cfg.nu
        s.max_iters, s.tol, s.norm = cfg.max_iters, cfg.tol, int(cfg.norm)
        s.initial_guess, s.seed, s.coarse_substeps = int(cfg.initial_guess), cfg.seed, cfg.coarse_substeps
        n = app.vector_size()
        functional = cfg.functional
        if isinstance(functional, str):
            if functional != "norm2":
                raise ConfigError(f"unknown functional {functional!r} (weights or 'norm2')")
            s.functional_kind, functional = 1, None  # ATM_FUNCTIONAL_NORM2
        for field, val in (("functional_w", functional), ("constant_value", cfg.constant_value),
                           ("provided", cfg.provided)):
            if val is not None:
                a = np.ascontiguousarray(val, np.float64).reshape(-1)
                if field == "provided" and a.size != hier.level(0).n_points * n:
                    raise ConfigError("provided initial guess has the wrong number of points")
                self._keep.append(a)
                setattr(s, field, ptr(a))
        rt = _capi.atm_runtime()
        rt.device, rt.n_shards, rt.world_size, rt.rank = device, workers, world_size, rank
        rt.trace = int(trace)
        rt.reuse_relax = int(reuse_relax)
        rt.storage = int(bool(cpoint_storage))  # ATM_STORE_CPOINTS
        rt.defer_guess = int(bool(defer_guess))
        rt.timeout_ms = int(timeout_ms)
        if nccl_id is not None:
            self._nid = C.create_string_buffer(bytes(nccl_id), 128)
            rt.nccl_id = C.cast(self._nid, C.c_void_p)
        h = C.c_void_p()
        st = lib().atm_create(C.byref(p), C.byref(g), C.byref(s), C.byref(rt), C.byref(h))
        if st != 0:
            _raise(st, lib().atm_create_error().decode())
        self._h = h
        self.n = lib().atm_vector_size(h)
        self.L = lib().atm_n_levels(h)

    def close(self):
        if getattr(self, "_h", None):
            lib().atm_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def _check(self, st):
        if st not in (0, 1):
            _raise(st, lib().atm_last_error(self._h).decode())
        return st

    # CycleDriver methods
    def setup(self):
        self._check(lib().atm_setup(self._h))

    def cycle(self):
        self._check(lib().atm_cycle(self._h))

    def nested_init(self):
        self._check(lib().atm_nested_init(self._h))

    def residual_norm(self) -> float:
        out = C.c_double()
        self._check(lib().atm_residual_norm(self._h, C.byref(out)))
        return out.value

    def drive(self) -> ConvergenceReport:
        norms = np.zeros(self.cfg.max_iters, np.float64)
        secs = np.zeros(self.cfg.max_iters, np.float64)
        rep = _capi.atm_report()
        st = lib().atm_solve(self._h, C.byref(rep), ptr(norms), ptr(secs))
        if st == 4:
            msg = lib().atm_last_error(self._h).decode()
            raise DivergenceError(rep.iterations, msg)
        self._check(st)
        t = self.timings()
        t["total"] = rep.total_seconds
        return ConvergenceReport(list(norms[: rep.iterations]), rep.iterations, bool(rep.converged),
                                 StopReason(rep.stop_reason), rep.total_seconds, rep.dof_steps, t,
                                 list(secs[: rep.iterations]))

    def iterate(self, count: int) -> np.ndarray:
        norms = np.zeros(count, np.float64)
        self._check(lib().atm_iterate(self._h, count, ptr(norms)))
        return norms

    def iterate_timed(self, count: int):
        """`count` cycles + norms; returns (norms, device milliseconds)."""
        norms = np.zeros(count, np.float64)
        ms = C.c_double()
        self._check(lib().atm_iterate_timed(self._h, count, ptr(norms), C.byref(ms)))
        return norms, ms.value

    def timings(self, with_counts: bool = False) -> dict:
        names = C.create_string_buffer(1024)
        secs = np.zeros(32, np.float64)
        k = lib().atm_phase_times(self._h, names, 1024, ptr(secs), 32)
        keys = names.value.decode().split(",") if k else []
        if not with_counts:
            return {key: float(secs[i]) for i, key in enumerate(keys)}
        cnt = (C.c_int * 32)()
        lib().atm_phase_counts(self._h, cnt, 32)
        return {key: (float(secs[i]), int(cnt[i])) for i, key in enumerate(keys)}

    def last_iteration_launches(self) -> int:
        n = C.c_int()
        lib().atm_last_iteration_stats(self._h, C.byref(n), None)
        return n.value

    # state access
    def level_points(self, l):
        return lib().atm_level_points(self._h, l)

    def get_level(self, level, which=0, first=0, count=None, out=None):
        npts = self.level_points(level)
        count = npts - first if count is None else count
        if out is None:
            out = np.zeros((count, self.n), np.float64)
        assert out.flags.c_contiguous and out.dtype == np.float64 and out.size == count * self.n
        self._check(lib().atm_get_level(self._h, level, which, first, count, ptr(out)))
        return out

    def set_level(self, level, values, which=0, first=0):
        a = np.ascontiguousarray(values, np.float64).reshape(-1, self.n)
        self._check(lib().atm_set_level(self._h, level, which, first, a.shape[0], ptr(a)))

    def state(self):
        return _StateView(self)

    # Application-level and kernel-level entry points
    def apply_phi(self, level, first_index, inputs):
        a = np.ascontiguousarray(inputs, np.float64).reshape(-1, self.n)
        out = np.empty_like(a)
        self._check(lib().atm_apply_phi(self._h, level, first_index, a.shape[0], ptr(a), ptr(out)))
        return out

    def forcing(self, level, first_index, count):
        out = np.empty((count, self.n), np.float64)
        self._check(lib().atm_forcing(self._h, level, first_index, count, ptr(out)))
        return out

    def inner_iterations(self) -> int:
        """Inner linear-solver iterations run so far (2D heat CG, Gray-Scott
        BiCGSTAB; 0 for the other families)."""
        v = C.c_ulonglong(0)
        self._check(lib().atm_inner_iterations(self._h, C.byref(v)))
        return int(v.value)

    def host_traffic(self):
        """(host-to-device, device-to-host) level-0 state bytes moved so far."""
        h, d = C.c_ulonglong(0), C.c_ulonglong(0)
        self._check(lib().atm_host_traffic(self._h, C.byref(h), C.byref(d)))
        return int(h.value), int(d.value)

    def f_relax(self, level, first_interval, count):
        self._check(lib().atm_kernel_f_relax(self._h, level, first_interval, count))

    def c_relax(self, level, first_c, count):
        self._check(lib().atm_kernel_c_relax(self._h, level, first_c, count))

    def residual(self, level, first, count):
        out = np.empty((count, self.n), np.float64)
        self._check(lib().atm_kernel_residual(self._h, level, first, count, ptr(out)))
        return out


@dataclasses.dataclass
class SolveResult:
    state: np.ndarray  # level-0 u, [n_points, n]
    report: ConvergenceReport
    driver: CycleDriver


def solve(app: Application, hier: Hierarchy, cfg: SolverConfig, **kw) -> SolveResult:
    """solve() (solver.hpp:134-135, solver.cpp:485-492) on the device."""
    drv = CycleDriver(app, hier, cfg, **kw)
    rep = drv.drive()
    return SolveResult(drv.get_level(0), rep, drv)


def run_parallel(app: Application, hier: Hierarchy, cfg: SolverConfig, workers: int, **kw):
    """runtime::run_parallel (parallel.hpp:26-27): `workers` time shards."""
    return solve(app, hier, cfg, workers=workers, **kw)


# ---------------------------------------------------------------------------
# host-only schedule helpers (no GPU needed)


def random_state(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, np.float64)
    lib().atm_random_state(C.c_uint64(seed), n, ptr(out))
    return out


# ---------------------------------------------------------------------------
# seeded synthetic inputs of the BASELINE configs 2-4 (pinned in DESIGN.md;
# SURVEY 8(d) leaves the mappings to the builder).  Host-side numpy, shared
# by the tests, the oracle runs and bench.py.


def gaussian_source(nx: int, seed: int = 11) -> np.ndarray:
    """Config 2: f(x, y) = sum_{j<8} a_j exp(-((x-x_j)^2 + (y-y_j)^2) / (2 s_j^2))
    on the nx x nx interior grid (x_i = (i+1) h, h = 1/(nx+1)), with
    (a, x, y, s)_j from random_state(seed, 32) mapped to a in [-1, 1),
    centres in [0.2, 0.8)^2, s in [0.03, 0.1)."""
    d = random_state(seed, 32).reshape(8, 4)
    h = 1.0 / (nx + 1)
    x = (np.arange(nx) + 1) * h
    X, Y = np.meshgrid(x, x, indexing="xy")  # row j = y index, column i = x index
    f = np.zeros((nx, nx))
    for a, cx, cy, s in d:
        cx, cy = 0.5 + 0.3 * cx, 0.5 + 0.3 * cy
        sig = 0.065 + 0.035 * s
        f += a * np.exp(-((X - cx) ** 2 + (Y - cy) ** 2) / (2.0 * sig * sig))
    return f.ravel()


def fourier_ic(nx: int, seed: int = 13) -> np.ndarray:
    """Config 4: u0 = sum_{p,q=1..8} c_pq sin(p pi x) sin(q pi y) / (p^2 + q^2),
    c_pq from random_state(seed, 64)."""
    c = random_state(seed, 64).reshape(8, 8)
    h = 1.0 / (nx + 1)
    x = (np.arange(nx) + 1) * h
    k = np.arange(1, 9)
    S = np.sin(np.pi * np.outer(k, x))          # [8, nx]
    w = c / (k[:, None] ** 2 + k[None, :] ** 2)  # w[p-1, q-1]
    u = S.T @ w.T @ S                           # u[j, i] = sum_pq w_pq sin(q pi y_j) sin(p pi x_i)
    return np.ascontiguousarray(u).ravel()


def allen_cahn_ic(n: int, seed: int = 3) -> np.ndarray:
    """Config 3: u0 = 0.05 random_state(seed, n), uniform in [-0.05, 0.05)."""
    return 0.05 * random_state(seed, n)


@dataclasses.dataclass
class RankLayout:
    workers: int
    fine_lo: list
    fine_hi: list
    coarse_lo: list
    coarse_hi: list


def build_layout(hier: Hierarchy, workers: int) -> RankLayout:
    g = hier.c_grid()
    arrs = [(C.c_int * max(workers, 1))() for _ in range(4)]
    st = lib().atm_build_layout(C.byref(g), workers, *arrs)
    if st != 0:
        _raise(st, lib().atm_create_error().decode())
    return RankLayout(workers, *[list(a) for a in arrs])


def rank_ranges(hier: Hierarchy, workers: int, rank: int) -> dict:
    g = hier.c_grid()
    L = hier.n_levels()
    arrs = [(C.c_int * L)() for _ in range(8)]
    st = lib().atm_rank_ranges(C.byref(g), workers, rank, *arrs)
    if st != 0:
        _raise(st, lib().atm_create_error().decode())
    keys = ["lo", "hi", "iv_first", "iv_count", "c_first", "c_count", "left_src", "right_dst"]
    return {k: list(a) for k, a in zip(keys, arrs)}


def window_recvs(hier: Hierarchy, workers: int, rank: int) -> list:
    g = hier.c_grid()
    cap = max(1, workers)  # at most one (src, first, count) triple per other rank
    buf = (C.c_int * (3 * cap))()
    n = lib().atm_window_recvs(C.byref(g), workers, rank, buf, cap)
    if n < 0:
        _raise(2, lib().atm_create_error().decode())
    if n > cap:
        raise RuntimeFault(f"window schedule has {n} sends, more than the {cap} ranks")
    return [(buf[3 * i], buf[3 * i + 1], buf[3 * i + 2]) for i in range(n)]


def build_comm_groups(n_coarse_points: int, k: int):
    """layout.cpp:65-81 (kept for schedule parity tests)."""
    if k < 1:
        raise ConfigError("comm groups: k must be at least 1")
    if n_coarse_points < 1:
        raise ConfigError("comm groups: empty coarse grid")
    first = [list(range(s, min(s + k, n_coarse_points))) for s in range(0, n_coarse_points, k)]
    second = []
    for s in range(k - 1, n_coarse_points, k):
        g = list(range(s, min(s + k, n_coarse_points)))
        if len(g) > 1:
            second.append(g)
    return first, second
