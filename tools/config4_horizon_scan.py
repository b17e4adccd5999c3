"""Config 4's spatial problem and time step (511^2, dt = 4/65536, four-level
FAS V-cycle m = (8, 8, 8), k = 2, random guess seed 20, tol 1e-10) solved to
tolerance over growing horizons N_t = 2048, 4096, 8192, ...: how the V-cycle
count grows with N_t (the full config is N_t = 65536).  One JSON line each.

  python tools/config4_horizon_scan.py 2048 4096 8192"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2107_09596_b200 as T  # noqa: E402

for nt in [int(a) for a in sys.argv[1:]]:
    app = T.Heat2D(511, folded=True, source=None, cg_rtol=1e-12, initial_condition=T.fourier_ic(511))
    hier = T.build_hierarchy(T.TimeGrid.make(0.0, 4.0 * nt / 65536, nt + 1), [8, 8, 8], 2)
    cfg = T.SolverConfig(mode=T.CycleMode.VCycle, relaxation=T.Relaxation.F, max_iters=200, tol=1e-10,
                         initial_guess=T.InitialGuess.Random, seed=20)
    drv = T.CycleDriver(app, hier, cfg, cpoint_storage=True)
    t0 = time.perf_counter()
    drv.setup()
    rep = drv.drive()
    secs = time.perf_counter() - t0
    print(json.dumps({"n_t": nt, "iterations": rep.iterations, "converged": bool(rep.converged),
                      "setup_to_tol_s": secs, "s_per_cycle": secs / max(rep.iterations, 1),
                      "history": [float(x) for x in rep.residual_norms]}), flush=True)
    drv.close()
