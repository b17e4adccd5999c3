"""Host<->device transfer rates of the e2e path: atm_setup (provided guess,
2D copy into the pitched level-0 array), atm_get_level (2D copy out), and
plain contiguous pinned copies (torch) for comparison."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2107_09596_b200 as T  # noqa: E402

n, npts = 4095, 2 ** 18 + 1
out = {}
g = np.random.default_rng(0).uniform(-1, 1, size=(npts, n))
o = np.empty_like(g)
assert T.lib().atm_host_register(g.ctypes.data, g.nbytes) == 0
assert T.lib().atm_host_register(o.ctypes.data, o.nbytes) == 0
app = T.Heat1D(n, manufactured_forcing=False, initial_condition=T.random_state(7, n))
hier = T.build_hierarchy(T.TimeGrid.make(0.0, 16.0, npts), [16], 8)
for cp in (False, True):
    cfg = T.SolverConfig(mode=T.CycleMode.TwoLevel, relaxation=T.Relaxation.F, tol=1e-300, max_iters=2,
                         initial_guess=T.InitialGuess.Provided, provided=g)
    drv = T.CycleDriver(app, hier, cfg, cpoint_storage=cp)
    t0 = time.perf_counter()
    drv.setup()
    t1 = time.perf_counter()
    drv.iterate(1)
    t2 = time.perf_counter()
    drv.get_level(0, out=o)
    t3 = time.perf_counter()
    out["cpoints" if cp else "full"] = dict(setup_s=t1 - t0, h2d_GBps=g.nbytes / (t1 - t0) / 1e9 / (16 if cp else 1),
                                            get_level_s=t3 - t2, d2h_GBps=o.nbytes / (t3 - t2) / 1e9)
    drv.close()
x = torch.from_numpy(g)  # registered above: pinned
d = torch.empty(g.shape, dtype=torch.float64, device="cuda")
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter(); d.copy_(x, non_blocking=True); torch.cuda.synchronize()
    t1 = time.perf_counter(); x.copy_(d, non_blocking=True); torch.cuda.synchronize(); t2 = time.perf_counter()
out["torch_contiguous"] = dict(h2d_GBps=g.nbytes / (t1 - t0) / 1e9, d2h_GBps=g.nbytes / (t2 - t1) / 1e9)
print(json.dumps(out))
