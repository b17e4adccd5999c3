"""BASELINE config 5 at full size: the batch-scaling sweep on one GPU.

1D heat, n = 4095, N_t = 2^18 on t in [0, 1], u0 = random_state(7, n),
random initial guess (seed 20), two-level AT-MGRIT with F-relaxation,
m in {16, 64} x k in {1, 2, 4, 8} plus k = N_T + 1 (the reference's classical
MGRIT global coarse grid), tol 1e-10 on the level-0 residual 2-norm.

Per (m, k):
  * time to tolerance: atm_setup + drive until the norm <= 1e-10, wall clock
    (one 8-byte norm readback per iteration), run with the bitwise-neutral
    opt-ins (relax reuse + C-point storage: same iterations, same norms as the
    default cycle -- tests/test_gpu_cpoints.py, test_relax_reuse_*);
  * device ms per iteration of the default cycle (CUDA events, 5 iterations
    after 2 warm-up) and of the opt-in cycle;
  * the final state at three time points against sequential time stepping
    (u_i = Phi(u_{i-1}) from u0: every converged run solves that space-time
    system, so the states agree to what the tolerance allows -- the
    size-independent check where the CPU reference cannot run in minutes).
  * with --cpu-rate R (the reference's DOF*steps/s from bench.py's
    cpu_baseline): its estimated time to tolerance, iterations x 2 n F_0 / R.

usage: python tools/config5_sweep.py [out.json] [--ms 16,64] [--ks 1,2,4,8,global]
"""
import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2107_09596_b200 as T  # noqa: E402

N, NPTS, TOL = 4095, 2 ** 18 + 1, 1e-10


def run(m, k, probe_rows):
    app = T.Heat1D(N, manufactured_forcing=False, initial_condition=T.random_state(7, N))
    n_c = (NPTS - 1) // m + 1
    kk = n_c if k == "global" else k
    hier = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, NPTS), [m], kk)
    # the front of the exact solution advances k coarse intervals per
    # iteration (test_solver.cpp:428-465): N_T / k iterations suffice
    max_iters = min(4 * (n_c - 1) // kk + 400, 50000)
    cfg = T.SolverConfig(mode=T.CycleMode.TwoLevel, relaxation=T.Relaxation.F, tol=TOL,
                         max_iters=max_iters, initial_guess=T.InitialGuess.Random, seed=20)
    out = dict(m=m, k=kk, k_label=str(k), n_coarse_points=n_c, max_iters=max_iters)

    # device ms per iteration: default cycle, then the opt-in cycle
    for name, kw in (("default", {}), ("reuse_cpoints", dict(reuse_relax=True, cpoint_storage=True))):
        drv = T.CycleDriver(app, hier, cfg, **kw)
        drv.setup()
        drv.iterate(2)
        _, ms = drv.iterate_timed(5)
        out[f"ms_per_iteration_{name}"] = ms / 5
        drv.close()

    drv = T.CycleDriver(app, hier, cfg, reuse_relax=True, cpoint_storage=True)
    t0 = time.perf_counter()
    drv.setup()
    rep = drv.drive()
    secs = time.perf_counter() - t0
    rows = {str(p): drv.get_level(0, first=p, count=1)[0] for p in probe_rows}
    drv.close()
    norms = rep.residual_norms
    out.update(iterations=rep.iterations, converged=bool(rep.converged),
               setup_to_tol_seconds=secs, first_norm=float(norms[0]), last_norm=float(norms[-1]),
               front_bound=math.ceil((n_c - 1) / kk))
    return out, rows


def sequential(probe_rows):
    """u_i = Phi(u_{i-1}) from u0 for all N_t steps: one interval (m = N_t),
    so one cycle's F-relaxation is exactly sequential time stepping."""
    app = T.Heat1D(N, manufactured_forcing=False, initial_condition=T.random_state(7, N))
    hier = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, NPTS), [NPTS - 1], 2)
    cfg = T.SolverConfig(mode=T.CycleMode.TwoLevel, relaxation=T.Relaxation.F, tol=1e-300, max_iters=1,
                         initial_guess=T.InitialGuess.Random, seed=20)
    drv = T.CycleDriver(app, hier, cfg)
    drv.setup()
    drv.iterate(1)
    rows = {p: drv.get_level(0, first=p, count=1)[0] for p in probe_rows}
    drv.close()
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out", nargs="?", default="gpurun_out/config5_sweep.json")
    ap.add_argument("--ms", default="16,64")
    ap.add_argument("--ks", default="1,2,4,8,global")
    ap.add_argument("--cpu-rate", type=float, default=None,
                    help="reference DOF*steps/s (bench.py cpu_baseline value)")
    args = ap.parse_args()
    probe_rows = [NPTS // 4, NPTS // 2, NPTS - 1]
    seq = sequential(probe_rows)
    res, states = [], {}
    for m in [int(x) for x in args.ms.split(",")]:
        for k in [x if x == "global" else int(x) for x in args.ks.split(",")]:
            r, rows = run(m, k, probe_rows)
            states[(m, str(k))] = rows
            res.append(r)
            print(json.dumps(r), flush=True)
    # every converged run solves the same space-time system as sequential
    # time stepping: compare the probe rows with it
    for key, r in zip(states, res):
        r["max_rel_err_vs_sequential"] = max(
            float(np.linalg.norm(states[key][str(p)] - seq[p]) / np.linalg.norm(seq[p])) for p in probe_rows)
        r["max_err_vs_sequential_over_u0"] = max(
            float(np.linalg.norm(states[key][str(p)] - seq[p]) / np.linalg.norm(T.random_state(7, N)))
            for p in probe_rows)
    if args.cpu_rate:
        for r in res:
            f0 = (NPTS - 1) - (NPTS - 1) // r["m"]
            r["reference_seconds_estimate"] = r["iterations"] * 2.0 * N * f0 / args.cpu_rate
    summary = dict(what=__doc__.split("\n\n")[0], n=N, n_points=NPTS, tol=TOL,
                   probe_rows=probe_rows, runs=res)
    os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
    json.dump(summary, open(args.out, "w"), indent=1)
    print(json.dumps(summary)[:4000])


if __name__ == "__main__":
    main()
