"""The paper's Gray-Scott experiment (table
tab:gray_two_level) on one B200: 128^2 periodic grid on [0, 2.5]^2,
F = 0.024, K = 0.06, Du = 8e-5, Dv = 4e-5, t in [0, 256] with 16 384 time
points, backward Euler + Newton (tol 1e-10), two-level AT-MGRIT with
F-relaxation, nested iterations, k = N_c / 2, stopping at space-time
residual 1e-7.  The reference's GrayScott Phi (gray_scott.cpp, inner
Jacobi-BiCGSTAB) is what runs; the paper used PETSc's Newton, so iteration
counts are compared, not times.  Prints one JSON object per m.

  python tools/gs_paper_probe.py [--m 512,256,128,64] [--out FILE]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_09596_b200 as T  # noqa: E402

PAPER = {512: (16, 12, 701.0, 165351.0), 256: (32, 10, 1167.0, 78230.0),
         128: (64, 9, 2022.0, 48675.0), 64: (128, 7, None, None)}
# tab:gray_three_level (256 processes, FCF): (m0, m1) -> (k, AT-MGRIT iterations,
# setup s, solve s, classical MGRIT iterations)
PAPER3 = {(64, 16): (8, 7, 2864.0, 41054.0, 7), (64, 8): (16, 7, 2174.0, 33688.0, 7),
          (64, 4): (32, 7, 2713.0, 34063.0, 7), (64, 2): (64, 7, 4247.0, 38571.0, 6)}


def run(ms, k, relax, classical=False):
    npts = 16384
    app = T.GrayScott(128)
    kk = k
    if classical:  # k = N_T + 1: the global coarse grid (classical MGRIT / Parareal)
        n = npts
        for f in ms:
            n = (n - 1) // f + 1
        kk = n + 1
    hier = T.build_hierarchy(T.TimeGrid.make(0.0, 256.0, npts), list(ms), kk)
    cfg = T.SolverConfig(mode=T.CycleMode.NestedV, relaxation=relax, tol=1e-7, max_iters=40)
    drv = T.CycleDriver(app, hier, cfg)
    drv.setup()
    t0 = time.perf_counter()
    drv.nested_init()
    t1 = time.perf_counter()
    norms = []
    while len(norms) < cfg.max_iters:
        norms.append(float(drv.iterate(1)[0]))
        if norms[-1] <= cfg.tol:
            break
    t2 = time.perf_counter()
    inner = drv.inner_iterations()
    drv.close()
    return dict(k=kk, iterations=len(norms), converged=norms[-1] <= cfg.tol, setup_s=t1 - t0,
                solve_s=t2 - t1, residual_norms=norms, bicgstab_iterations=inner)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", default="512,256,128,64")
    ap.add_argument("--three", action="store_true", help="tab:gray_three_level (FCF) instead")
    ap.add_argument("--classical", action="store_true", help="also k = N_T + 1 (MGRIT) for --three")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    res = []
    def safe(*args, **kw):
        try:
            return run(*args, **kw)
        except T.api.TempoError as e:  # e.g. the reference's Newton failing on a dt = 16 coarse step
            return dict(error=f"{type(e).__name__}: {e}")

    if a.three:
        for (m0, m1), (k, it, su, so, it_mgrit) in PAPER3.items():
            r = dict(m=[m0, m1], relaxation="FCF", **safe((m0, m1), k, T.Relaxation.FCF),
                     paper_iterations=it, paper_setup_s=su, paper_solve_s=so)
            print(json.dumps(r), flush=True)
            res.append(r)
            if a.classical:
                r = dict(m=[m0, m1], relaxation="FCF", variant="classical MGRIT (k = N_T + 1)",
                         **safe((m0, m1), k, T.Relaxation.FCF, classical=True), paper_iterations=it_mgrit)
                print(json.dumps(r), flush=True)
                res.append(r)
        if a.out:
            json.dump(res, open(a.out, "w"), indent=1)
        return
    for m in [int(v) for v in a.m.split(",")]:
        npts = 16384
        nc = (npts - 1) // m + 1
        k = max(1, (npts // m) // 2)
        app = T.GrayScott(128)
        hier = T.build_hierarchy(T.TimeGrid.make(0.0, 256.0, npts), [m], k)
        cfg = T.SolverConfig(mode=T.CycleMode.NestedV, relaxation=T.Relaxation.F, tol=1e-7, max_iters=40)
        drv = T.CycleDriver(app, hier, cfg)
        drv.setup()
        t0 = time.perf_counter()
        drv.nested_init()  # the paper's "setup": nested iteration
        t1 = time.perf_counter()
        norms = []
        while len(norms) < cfg.max_iters:  # drive(): cycle + stopping norm
            norms.append(float(drv.iterate(1)[0]))
            if norms[-1] <= cfg.tol:
                break
        t2 = time.perf_counter()
        inner = drv.inner_iterations()
        drv.close()
        p = PAPER.get(m)
        r = dict(m=m, k=k, coarse_points=nc, iterations=len(norms), converged=norms[-1] <= cfg.tol,
                 setup_s=t1 - t0, solve_s=t2 - t1, residual_norms=norms,
                 bicgstab_iterations=inner,
                 paper_iterations=p[1] if p else None, paper_setup_s=p[2] if p else None,
                 paper_solve_s=p[3] if p else None)
        print(json.dumps(r), flush=True)
        res.append(r)
    if a.out:
        json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
