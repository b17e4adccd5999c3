"""Full-size golden fixtures for BASELINE configs 2, 3 and 4 from the COMPILED
REFERENCE's own cycle driver (oracle/_ref/tempo_ref: `runtime::run_parallel`
over all host threads, /root/reference/proj/src/parallel.cpp:331-405).  The
reference has no Phi for these problems, so tempo_ref's `OracleApp` supplies
the restated Phi (oracle/atm_oracle.c: h2_solve / ac_step) through the
reference's Application interface (application.hpp:33-76); the cycles --
relaxation, restriction, truncated windows, FAS, correction, norm, stopping
-- are the reference's (solver.cpp:152-435).

Each fixture holds the iteration count and residual history to tol 1e-10 and
every SAMPLE-th level-0 row of the final state plus its 2-norm (the full state
is 0.5 GB and up): tests/test_gpu_fullsize.py compares the device solve
against them.  A Newton-cap failure (NonlinearSolveError, gray_scott.cpp:
165-169) is recorded with the failing cycle and the history before it: a
first run names the failing cycle (tempo_ref reports the last iteration a
phase ran in), a second run with max_iters = that cycle - 1 yields the history.

  python tests/golden/make_fullsize.py TAG [TAG ...]
      TAG in config2, config3, config3_constant, config3_newton1e-11, config4s

Config definitions follow DESIGN.md section 9 (pinned choices).  config4s is
BASELINE config 4's spatial problem and time step (511^2, dt = 4/65536,
four-level FAS V-cycle m = (8, 8, 8), k = 2) over a short horizon (2048 steps:
levels of 2049, 257, 33, 5 points -- run_parallel takes at most 5 workers)
so the CPU reference finishes in about an hour; its rows keep every 16th
unknown (a 511^2 state is 2 MB).
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

TOL = 1e-10


def gaussian_source(nx):
    # same construction as paper_2107_09596_b200.gaussian_source (DESIGN 9)
    import paper_2107_09596_b200 as T
    return T.gaussian_source(nx)


def fourier_ic(nx):
    import paper_2107_09596_b200 as T
    return T.fourier_ic(nx)


def config(tag):
    """(meta, tempo_ref args, input files) for one fixture tag."""
    if tag == "config2":
        nx = 127
        return (dict(config=2, guess="random", sample_every=256),
                dict(problem="heat2d", nx=nx, folded=0, cg_rtol=1e-12, cg_max=10000, tf=1.0,
                     n_points=4097, m=16, k=4, mode="two-level", guess="random", seed=20,
                     max_iters=200, tol=TOL),
                dict(source_file=gaussian_source(nx)))
    if tag.startswith("config3"):
        guess = "constant" if "constant" in tag else "random"
        ntol = float(tag.split("newton")[1]) if "newton" in tag else 1e-12
        meta = dict(config=3, guess=guess, sample_every=1024)
        if ntol != 1e-12:
            meta["newton_tol"] = ntol
        return (meta,
                dict(problem="allen_cahn", n=4096, eps=0.02, length=1.0, newton_tol=ntol,
                     newton_max=30, tf=8.0, n_points=16385, m="8,8", k=4, mode="v-cycle",
                     guess=guess, seed=20, max_iters=200, tol=TOL),
                dict(ic_file=0.05 * O.random_state(3, 4096)))
    if tag == "config4s":
        nx = 511
        return (dict(config=4, guess="random", sample_every=256, dof_stride=16, n_points=2049, tf=0.125),
                dict(problem="heat2d", nx=nx, folded=1, cg_rtol=1e-12, cg_max=100000,
                     tf=2048 * 4.0 / 65536, n_points=2049, m="8,8,8", k=2, mode="v-cycle",
                     guess="random", seed=20, max_iters=60, tol=TOL),
                dict(ic_file=fourier_ic(nx)))
    raise SystemExit(f"unknown tag {tag}")


def main(tags):
    for tag in tags:
        meta, args, files = config(tag)
        args = dict(args, workers=0)  # all host threads
        meta.update(tol=TOL, generator="tempo_ref run_parallel (reference CycleDriver, restated Phi)")
        t0 = time.time()
        res, u = O.run_ref(args, out_u=True, files=files, timeout=6 * 3600)
        if "error" in res:
            if res["error"] not in ("nonlinear", "runtime") or "Newton" not in res.get("what", ""):
                raise SystemExit(f"{tag}: {res}")
            failed = int(res["last_iteration"])
            hist, _ = O.run_ref(dict(args, max_iters=failed - 1), files=files, timeout=6 * 3600)
            assert "error" not in hist and len(hist["history"]) == failed - 1, hist
            meta.update(error=res["what"], code=5, failed_at_iteration=failed,
                        history=[float(x) for x in hist["history"]],
                        ref_seconds=time.time() - t0, workers=hist["workers"])
        else:
            n = u.size // int(args["n_points"])
            u = u.reshape(int(args["n_points"]), n)
            ds = meta.get("dof_stride", 1)
            np.save(os.path.join(HERE, f"fullsize_{tag}_rows.npy"), u[::meta["sample_every"], ::ds].copy())
            meta.update(iterations=int(res["iterations"]), converged=bool(res["converged"]),
                        history=[float(x) for x in res["history"]],
                        state_l2=float(np.linalg.norm(u)), ref_seconds=res["seconds"],
                        workers=res["workers"])
        with open(os.path.join(HERE, f"fullsize_{tag}.json"), "w") as f:
            json.dump(meta, f, indent=1)
        print(json.dumps({k: v for k, v in meta.items() if k != "history"}), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
