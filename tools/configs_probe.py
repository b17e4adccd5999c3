"""Device throughput of the BASELINE configs 1-4 (the parity configs; config 5
is bench.py's workload).  Per config: build, setup (+ nested init), one
warm-up iteration, then K timed iterations with CUDA events
(CycleDriver.iterate_timed).  DOF*steps counts n x relaxation Phi
applications (2 F-sweeps per level visit, + the C-relaxation for FCF), the
same count atm_solve reports.  Writes one JSON object per config.

  python tools/configs_probe.py [--out profiles/configs_r01.json] [--only 2,3]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2107_09596_b200 as T  # noqa: E402


def configs():
    c = {}
    # 1: 1D heat nx=63, Nt=1024, two-level m=16 k=2 FCF
    c[1] = dict(
        name="config1_heat1d_n63_Nt1024_m16_k2_FCF",
        app=lambda: T.Heat1D(63, 0.0, 1.0, folded=False, manufactured_forcing=False,
                             initial_condition=np.sin(np.pi * np.arange(1, 64) / 64) + 0.1 * T.random_state(1, 63)),
        grid=(0.0, 1.0, 1025, [16], 2), mode=T.CycleMode.TwoLevel, relax=T.Relaxation.FCF, iters=10)
    # 2: 2D heat 127^2, Nt=4096 over [0,1], Gaussian source, two-level m=16 k=4
    c[2] = dict(
        name="config2_heat2d_127x127_Nt4096_m16_k4",
        app=lambda: T.Heat2D(127, folded=False, source=T.gaussian_source(127), cg_rtol=1e-12),
        grid=(0.0, 1.0, 4097, [16], 4), mode=T.CycleMode.TwoLevel, relax=T.Relaxation.F, iters=2)
    # 3: Allen-Cahn n=4096, Nt=16384 over [0,8], three-level m=8 k=4 (FAS)
    c[3] = dict(
        name="config3_allencahn_n4096_Nt16384_m8x8_k4",
        app=lambda: T.AllenCahn(4096, 0.02, 1.0, 1e-12, 30, initial_condition=T.allen_cahn_ic(4096)),
        grid=(0.0, 8.0, 16385, [8, 8], 4), mode=T.CycleMode.VCycle, relax=T.Relaxation.F, iters=2)
    # 4: 2D heat 511^2, four-level m=8 k=2 (FAS), Fourier u0.  Full N_t = 65536
    # needs ~205 GB of level arrays (more than one B200): N_t = 4096 here
    c[4] = dict(
        name="config4_heat2d_511x511_Nt4096(of 65536)_m8x8x8_k2",
        app=lambda: T.Heat2D(511, folded=True, source=None, cg_rtol=1e-12,
                             initial_condition=T.fourier_ic(511)),
        grid=(0.0, 4.0 * 4096 / 65536, 4097, [8, 8, 8], 2), mode=T.CycleMode.VCycle, relax=T.Relaxation.F,
        iters=1)
    # 4 at the full N_t = 65536 on one GPU: level 0 with C-point storage
    # (17 GB instead of 137 GB; ~95 GB of level arrays in all); one cycle
    c[7] = dict(
        name="config4_heat2d_511x511_Nt65536_m8x8x8_k2_cpoint_storage",
        app=lambda: T.Heat2D(511, folded=True, source=None, cg_rtol=1e-12,
                             initial_condition=T.fourier_ic(511)),
        grid=(0.0, 4.0, 65537, [8, 8, 8], 2), mode=T.CycleMode.VCycle, relax=T.Relaxation.F,
        iters=1, warm=0, cpts=True)
    # Gray-Scott desk run (configs/grayscott_desk.cfg; the paper's flagship
    # problem): n = 32, 512 points over [0, 64], nested-v, m = k = 16
    c[6] = dict(
        name="grayscott_desk_n32_512pts_m16_k16_nested",
        app=lambda: T.GrayScott(32),
        grid=(0.0, 64.0, 512, [16], 16), mode=T.CycleMode.NestedV, relax=T.Relaxation.F, iters=2,
        guess=T.InitialGuess.Constant, tol=1e-7)
    return c


def dof_steps(hier, n, relax, nu=1, reuse=False):
    tot = 0.0
    for l in range(hier.n_levels() - 1):
        np_l = hier.level(l).n_points
        nc = (np_l - 1) // hier.m[l] + 1
        F = np_l - nc
        # relax reuse: the level-0 opening F-sweep is not run
        per = F if (reuse and l == 0 and relax == T.Relaxation.F) else 2.0 * F
        if relax == T.Relaxation.FCF:
            per += nu * (F + nc - 1)
        tot += per * n
    return tot


def run(cfg, reuse=False):
    app = cfg["app"]()
    t0, tf, npts, ms, k = cfg["grid"]
    hier = T.build_hierarchy(T.TimeGrid.make(t0, tf, npts), ms, k)
    sc = T.SolverConfig(mode=cfg["mode"], relaxation=cfg["relax"], max_iters=100, tol=cfg.get("tol", 1e-10),
                        initial_guess=cfg.get("guess", T.InitialGuess.Random), seed=20)
    reuse = reuse and cfg["relax"] == T.Relaxation.F
    drv = T.CycleDriver(app, hier, sc, cpoint_storage=cfg.get("cpts", False), reuse_relax=reuse)
    w0 = time.perf_counter()
    drv.setup()
    if cfg["mode"] == T.CycleMode.NestedV:
        drv.nested_init()
    drv.iterate(max(cfg.get("warm", 1), 1) if reuse else cfg.get("warm", 1))
    setup_s = time.perf_counter() - w0
    it0 = drv.inner_iterations()
    norms, ms_dev = drv.iterate_timed(cfg["iters"])
    inner = drv.inner_iterations() - it0
    ds = dof_steps(hier, app.vector_size(), cfg["relax"], reuse=reuse) * cfg["iters"]
    r = dict(config=cfg["name"] + ("+relax_reuse" if reuse else ""), n=app.vector_size(), iterations_timed=cfg["iters"],
             ms_per_iteration=ms_dev / cfg["iters"], dof_steps_per_s=ds / (ms_dev * 1e-3),
             setup_plus_first_iteration_s=setup_s, norms=[float(v) for v in norms])
    if inner:
        # SURVEY 8(d) second unit for the inner-solver configs: DOF x CG
        # iterations per second, and the 2-pass fused-CG floor of 64 B per
        # DOF per CG iteration against the measured HBM peak
        rate = app.vector_size() * inner / (ms_dev * 1e-3)
        r.update(inner_iterations=inner, dof_inner_iterations_per_s=rate,
                 cg_2pass_equiv_GBps=64.0 * rate / 1e9, cg_2pass_equiv_frac_of_hbm=64.0 * rate / 6534.5e9)
    return r


# bounded CPU samples (C oracle restatement, one thread) of the same n and
# per-level dt at reduced N_t: one cycle each
# (config 4: two levels, m = 8, at 17 points -- its four-level hierarchy
# needs >= 513 points, hours of single-thread CG)
CPU_SAMPLES = {1: (1025, None), 2: (257, None), 3: (1025, None), 4: (17, [8]), 6: (512, None)}


def run_cpu(i, cfg):
    from oracle import oracle as O
    app = cfg["app"]()
    t0, tf, npts, ms, k = cfg["grid"]
    sp, ms_over = CPU_SAMPLES[i]
    if ms_over:
        ms = ms_over
    tf_s = t0 + (tf - t0) * (sp - 1) / (npts - 1)
    hier = T.build_hierarchy(T.TimeGrid.make(t0, tf_s, sp), ms, k)
    keep = []
    p = app.c_problem(keep)
    kind = {T.Heat1D: O.HEAT1D, T.Heat2D: O.HEAT2D, T.AllenCahn: O.ALLEN_CAHN,
            T.GrayScott: O.GRAY_SCOTT}[type(app)]
    prob = dict(kind=kind, n=app.vector_size(), folded=int(p.folded), manufactured=int(p.manufactured),
                eps=p.eps, length=p.length, newton_tol=p.newton_tol, newton_max=p.newton_max,
                nx=p.nx, cg_rtol=p.cg_rtol, cg_max=p.cg_max,
                source=getattr(app, "source", None), ic=getattr(app, "ic", None))
    mode = {T.CycleMode.TwoLevel: O.TWO_LEVEL, T.CycleMode.VCycle: O.VCYCLE,
            T.CycleMode.NestedV: O.NESTED_V}[cfg["mode"]]
    if len(ms) == 1 and mode == O.VCYCLE:
        mode = O.VCYCLE  # FAS two-grid (folded)
    orc = O.Driver(prob, dict(t0=t0, tf=tf_s, n_points=sp, m=list(ms), k=k),
                   dict(mode=mode, relaxation=O.RELAX_FCF if cfg["relax"] == T.Relaxation.FCF else O.RELAX_F,
                        max_iters=100, tol=cfg.get("tol", 1e-10),
                        initial_guess=O.GUESS_CONSTANT if cfg.get("guess") == T.InitialGuess.Constant
                        else O.GUESS_RANDOM, seed=20))
    orc.setup()
    if mode == O.NESTED_V:
        orc.nested_init()
    w0 = time.perf_counter()
    orc.cycle()
    dt = time.perf_counter() - w0
    ds = dof_steps(hier, app.vector_size(), cfg["relax"])
    return dict(cpu_kind="port (oracle/atm_oracle.c, 1 thread)", cpu_sample_points=sp, cpu_sample_m=list(ms),
                cpu_s_per_iteration=dt, cpu_dof_steps_per_s=ds / dt)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--only", default="1,2,3,4,6")
    ap.add_argument("--cpu", action="store_true")
    ap.add_argument("--reuse", action="store_true",
                    help="opt-in relax reuse (skip the level-0 opening F-sweep; bitwise the same cycles)")
    a = ap.parse_args()
    res = []
    cs = configs()
    for i in [int(x) for x in a.only.split(",")]:
        r = run(cs[i], a.reuse)
        if a.cpu:
            r.update(run_cpu(i, cs[i]))
        print(json.dumps(r), flush=True)
        res.append(r)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
