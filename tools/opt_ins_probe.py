"""Config 5 (bench workload) device ms per iteration with the opt-ins:
full storage, relax reuse, relax reuse + C-point storage (CUDA events,
CycleDriver.iterate_timed, after 2 warm-up iterations)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2107_09596_b200 as T  # noqa: E402

n, npts, K = 4095, 2 ** 18 + 1, 10
app = T.Heat1D(n, manufactured_forcing=False, initial_condition=T.random_state(7, n))
hier = T.build_hierarchy(T.TimeGrid.make(0.0, 16.0, npts), [16], 8)
cfg = T.SolverConfig(mode=T.CycleMode.TwoLevel, relaxation=T.Relaxation.F, tol=1e-300, max_iters=100,
                     initial_guess=T.InitialGuess.Random, seed=20)
out = {}
ref = None
for name, kw in [("full", {}), ("reuse", dict(reuse_relax=True)),
                 ("reuse+cpoints", dict(reuse_relax=True, cpoint_storage=True))]:
    drv = T.CycleDriver(app, hier, cfg, **kw)
    drv.setup()
    drv.iterate(2)
    norms, ms = drv.iterate_timed(K)
    if ref is None:
        ref = norms
    out[name] = dict(ms_per_iteration=ms / K, same_norms=bool(np.array_equal(norms, ref)))
    drv.close()
print(json.dumps(out))
