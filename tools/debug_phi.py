import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2107_09596_b200 as T
from helpers import device_objects, oracle_driver
from oracle import oracle as O
for n, tf, npts, level in [(4095, 0.25, 4097, 0), (4095, 0.25, 4097, 1), (4096, 1.0, 33, 1), (4095, 1.0/64, 4097, 1)]:
    args = dict(problem="heat1d", n=n, tf=tf, n_points=npts, m=16 if npts > 33 else 4, k=8, manufactured=0, guess="random", seed=5, max_iters=5, tol=1e-9, substeps=1)
    app, hier, cfg = device_objects(args)
    drv = T.CycleDriver(app, hier, cfg); orc = oracle_driver(args)
    x = O.random_state(300, n)[None, :]
    got = drv.apply_phi(level, 1, x)[0]; want = orc.step(level, 1, x[0])
    err = np.abs(got - want) / np.abs(want).max()
    blocks = [float(err[i:i+512].max()) for i in range(0, n, 512)]
    print(n, tf, level, "max rel", err.max(), "per-warp", ["%.0e" % b for b in blocks])
