"""Generate golden fixtures from the COMPILED REFERENCE (oracle/_ref/tempo_ref,
built by oracle/Makefile from /root/reference/proj/src in place).

Run in the dev container (where /root/reference exists):
    python tests/golden/make_golden.py
Writes tests/golden/cases.json (+ small .npy arrays).  Inputs (initial
conditions) are generated with the reference's own splitmix64 random_state,
restated bitwise in oracle/atm_oracle.c, and stored next to the outputs.
"""
from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402


def sin_profile(n, x0=0.0, x1=1.0):
    h = (x1 - x0) / (n + 1)
    return np.array([math.sin(3.14159265358979323846 * (x0 + h * (i + 1))) for i in range(n)])


def ic_config1():
    # BASELINE config 1 pinned in SURVEY 8(d): sin(pi x) + 0.1 * random_state(1, 63)
    return sin_profile(63) + 0.1 * O.random_state(1, 63)


def ic_config5(n=4095):
    # BASELINE config 5: seeded random u0 = random_state(7, n)
    return O.random_state(7, n)


# store_u: True = the whole final level-0 state; an int s > 1 = every s-th
# point row (plus the last) -- the final-state bar at sizes too large to commit.
CASES = {
    # name: (args, ic-array-or-None, store_u)
    "config1": (dict(problem="heat1d", n=63, tf=1.0, n_points=1025, m=16, k=2, relax="FCF",
                     tol=1e-10, manufactured=0, guess="random", seed=20, max_iters=100, workers=1),
                ic_config1, True),
    "heat_full_single": (dict(problem="heat1d", n=1025, tf=3.0, n_points=16384, m=128, k=12,
                              tol=1e-7, guess="random", seed=20, max_iters=200, workers=8),
                         None, 1024),
    "dahlquist_cfg": (dict(problem="dahlquist", **{"lambda": -1.0}, tf=2.0, n_points=33, m=4, k=3,
                           tol=1e-9, guess="random", seed=11, max_iters=40, workers=1), None, True),
    "heat_det_65": (dict(problem="heat1d", n=65, tf=3.0, n_points=257, m=16, k=5, tol=1e-8,
                         guess="random", seed=71, max_iters=40, workers=1), None, True),
    "heat_fas_nested_fcf": (dict(problem="heat1d", n=33, folded=1, tf=3.0, n_points=129, m="4,4",
                                 k=3, mode="nested-v", relax="FCF", guess="random", seed=3,
                                 tol=1e-9, max_iters=30, workers=1), None, True),
    "heat_fas_vcycle_f": (dict(problem="heat1d", n=47, folded=1, tf=2.0, n_points=257, m="4,4",
                               k=4, mode="v-cycle", guess="random", seed=5, tol=1e-9,
                               max_iters=40, substeps=2, workers=1), None, True),
}
for k in (2, 4, 8, 12, 64, 128):
    CASES[f"kstudy_k{k}"] = (dict(problem="heat1d", n=1025, tf=3.0, n_points=16384, m=128, k=k,
                                  tol=1e-7, guess="random", seed=20, max_iters=300, workers=8),
                             None, 1024)
# FunctionalChange stopping norm (solver.cpp:380-396): the reference CLI's
# functional u.norm2() (run_config.cpp:241-243) and a linear functional w.u
W65 = lambda: O.random_state(5, 65)  # noqa: E731
CASES["functional_norm2"] = (dict(problem="heat1d", n=65, tf=3.0, n_points=257, m=16, k=5, tol=1e-9,
                                  guess="random", seed=71, max_iters=40, workers=1, norm="functional",
                                  functional="norm2"), None, True)
CASES["functional_weights"] = (dict(problem="heat1d", n=65, tf=3.0, n_points=257, m=16, k=5, tol=1e-9,
                                    guess="random", seed=71, max_iters=40, workers=1, norm="functional",
                                    functional="weights"), None, True, dict(w_file=W65))
CASES["functional_norm2_5r"] = (dict(problem="heat1d", n=4095, tf=1.0, n_points=4097, m=16, k=8,
                                     tol=1e-10, manufactured=0, guess="random", seed=20, max_iters=200,
                                     workers=8, norm="functional", functional="norm2"), ic_config5, 256)

# BASELINE config 5 shape at N_t = 2^14: m in {16, 64}, k in
# {1, 2, 4, 8} plus classical k = N_T + 1; max_iters = 2 N_T / k + 50.
for m in (16, 64):
    n_t = 16384 // m
    for k in (1, 2, 4, 8, n_t + 1):
        name = f"config5r_k{k}" if m == 16 else f"config5r_m{m}_k{k}"
        CASES[name] = (dict(problem="heat1d", n=4095, tf=1.0, n_points=16385, m=m, k=k,
                            tol=1e-10, manufactured=0, guess="random", seed=20,
                            max_iters=max(400, 2 * n_t // k + 50), workers=8), ic_config5, 256)


def main(only=None):
    out_path = os.path.join(HERE, "cases.json")
    db = json.load(open(out_path)) if os.path.exists(out_path) else {}
    for name, spec in CASES.items():
        args, icf, store_u = spec[:3]
        if only and name not in only:
            continue
        files = {}
        for key, fn in (spec[3] if len(spec) > 3 else {}).items():
            files[key] = fn()
            np.save(os.path.join(HERE, f"{name}_{key}.npy"), files[key])
        if icf is not None:
            ic = icf()
            files["ic_file"] = ic
            np.save(os.path.join(HERE, f"{name}_ic.npy"), ic)
        res, u = O.run_ref(args, out_u=True, files=files, timeout=7200)
        if "error" in res:
            raise SystemExit(f"{name}: {res}")
        n = int(args.get("n", 1)) if args["problem"] == "heat1d" else 1
        u = u.reshape(-1, n)
        entry = dict(args=args, iterations=res["iterations"], converged=res["converged"],
                     history=res["history"], ref_seconds=res["seconds"],
                     u_l2=float(np.sqrt(np.sum(u * u))), u_last=u[-1].tolist()[:8],
                     has_ic=icf is not None)
        if store_u is True:
            np.save(os.path.join(HERE, f"{name}_u.npy"), u)
        elif store_u:
            idx = sorted(set(range(0, u.shape[0], store_u)) | {u.shape[0] - 1})
            np.save(os.path.join(HERE, f"{name}_rows.npy"), u[idx])
            entry["row_stride"] = int(store_u)
        entry["store_u"] = store_u is True
        db[name] = entry
        print(f"{name}: iterations={res['iterations']} converged={res['converged']} "
              f"({res['seconds']:.2f} s)", flush=True)
        json.dump(db, open(out_path, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1:] or None)
