"""A/B helper: config-5 device ms per iteration and phase split for the
library named by ATM_LIB (default: the in-tree build)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_09596_b200 as T  # noqa: E402

n, npts, K = 4095, 2 ** 18 + 1, 10
app = T.Heat1D(n, manufactured_forcing=False, initial_condition=T.random_state(7, n))
hier = T.build_hierarchy(T.TimeGrid.make(0.0, float(os.environ.get("AB_TF", "1.0")), npts), [16], 8)
cfg = T.SolverConfig(mode=T.CycleMode.TwoLevel, relaxation=T.Relaxation.F, tol=1e-300, max_iters=100,
                     initial_guess=T.InitialGuess.Random, seed=20)
drv = T.CycleDriver(app, hier, cfg)
drv.setup()
drv.iterate(2)
best = 1e9
for _ in range(3):
    norms, ms = drv.iterate_timed(K)
    best = min(best, ms / K)
drv.close()
tr = T.CycleDriver(app, hier, cfg, trace=True)
tr.setup()
tr.iterate(3)
ph = {k: round(v * 1e3 / 3, 4) for k, v in tr.timings().items()}
print(json.dumps({"lib": os.environ.get("ATM_LIB", "in-tree"), "ms_per_iteration": best,
                  "last_norm": float(norms[-1]), "phase_ms": ph}))
