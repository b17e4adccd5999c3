"""Full-size golden fixtures for BASELINE configs 2 and 3 from the C oracle
restatement (oracle/atm_oracle.c; single-threaded, minutes to an hour per
config on the dev container).  Each fixture holds the oracle's iteration
count and residual history to tol 1e-10 and every SAMPLE-th level-0 row of
its final state (the full state is 0.5 GB): tests/test_gpu_fullsize.py
compares the device solve against them.

  python tests/golden/make_fullsize.py {2,3} [random|constant] [newton_tol (config 3, default 1e-12)]

Config definitions follow DESIGN.md section 9 (pinned choices)."""
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
SAMPLE = {2: 256, 3: 1024}


def gaussian_source(nx):
    # same construction as paper_2107_09596_b200.gaussian_source (DESIGN 9)
    import paper_2107_09596_b200 as T
    return T.gaussian_source(nx)


def config(c, guess="random", newton_tol=1e-12):
    if c == 2:
        nx = 127
        return (dict(kind=O.HEAT2D, n=nx * nx, nx=nx, folded=0, source=gaussian_source(nx), ic=None,
                     cg_rtol=1e-12, cg_max=10000),
                dict(tf=1.0, n_points=4097, m=[16], k=4),
                dict(mode=O.TWO_LEVEL, relaxation=O.RELAX_F, max_iters=200, tol=TOL,
                     initial_guess=O.GUESS_RANDOM, seed=20))
    if c == 3:
        n = 4096
        return (dict(kind=O.ALLEN_CAHN, n=n, eps=0.02, length=1.0, newton_tol=newton_tol, newton_max=30,
                     folded=1, ic=0.05 * O.random_state(3, n)),
                dict(tf=8.0, n_points=16385, m=[8, 8], k=4),
                dict(mode=O.VCYCLE, relaxation=O.RELAX_F, max_iters=200, tol=TOL,
                     initial_guess=O.GUESS_RANDOM if guess == "random" else O.GUESS_CONSTANT,
                     seed=20))
    raise SystemExit(f"unknown config {c}")


def main():
    c = int(sys.argv[1])
    guess = sys.argv[2] if len(sys.argv) > 2 else "random"
    ntol = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-12
    tag = f"config{c}" + ("" if guess == "random" else f"_{guess}") + ("" if ntol == 1e-12 else f"_newton{ntol:g}")
    p, g, s = config(c, guess, ntol)
    t0 = time.time()
    d = O.Driver(p, g, s)
    meta = dict(config=c, guess=guess, tol=TOL, newton_tol=ntol, sample_every=SAMPLE[c])
    try:
        res = d.drive()
    except O.OracleError as e:
        # the reference's failure behaviour is part of the contract (Newton
        # cap -> NonlinearSolveError, gray_scott.cpp:165-169): record the
        # failing iteration and the history before it
        meta.update(error=str(e), code=int(e.code),
                    failed_at_iteration=int(e.iterations) + 1,
                    history=[float(x) for x in e.history], oracle_seconds=time.time() - t0)
        with open(os.path.join(HERE, f"fullsize_{tag}.json"), "w") as f:
            json.dump(meta, f, indent=1)
        print(json.dumps({k: v for k, v in meta.items() if k != "history"}))
        return
    u = d.array(0)
    np.save(os.path.join(HERE, f"fullsize_{tag}_rows.npy"), u[::SAMPLE[c]].copy())
    meta.update(iterations=int(res["iterations"]), converged=bool(res["converged"]),
                history=[float(x) for x in res["history"]], state_l2=float(np.linalg.norm(u)),
                oracle_seconds=time.time() - t0)
    with open(os.path.join(HERE, f"fullsize_{tag}.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(json.dumps({k: v for k, v in meta.items() if k != "history"}))


if __name__ == "__main__":
    main()
