import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2107_09596_b200 as T
from helpers import device_objects, oracle_driver, rel_l2
for n in (2049, 2100, 3001):
    args = dict(problem="heat1d", n=n, tf=0.25, n_points=257, m=8, k=4, manufactured=1,
                guess="random", seed=13, max_iters=60, tol=1e-9)
    app, hier, cfg = device_objects(args)
    drv = T.CycleDriver(app, hier, cfg); drv.setup()
    orc = oracle_driver(args); orc.setup()
    print(n, 'init', np.array_equal(drv.get_level(0), orc.array(0)))
    drv.f_relax(0, 0, 32); orc.f_relax(0, 0, 32)
    print(n, 'f_relax', rel_l2(drv.get_level(0), orc.array(0)))
    r1 = drv.residual(0, 0, 257); r2 = orc.residual(0, 0, 257)
    print(n, 'resid', np.max(np.abs(r1 - r2)))
    d2 = T.CycleDriver(app, hier, cfg); d2.setup(); o2 = oracle_driver(args); o2.setup()
    d2.cycle(); o2.cycle()
    print(n, 'cycle u', rel_l2(d2.get_level(0), o2.array(0)), 'r1', rel_l2(d2.get_level(1, 3), o2.array(1, 'r')))
