import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2107_09596_b200 as T
from helpers import device_objects, oracle_driver, rel_l2
from oracle import oracle as O
n, npts = 4095, 4097
ic = O.random_state(7, n)
args = dict(problem="heat1d", n=n, tf=1.0, n_points=npts, m=16, k=int(sys.argv[1]) if len(sys.argv) > 1 else 8,
            manufactured=0, guess="random", seed=20, tol=1e-10, max_iters=2)
app, hier, cfg = device_objects(args, ic=ic)
drv = T.CycleDriver(app, hier, cfg); drv.setup()
orc = oracle_driver(args, ic=ic); orc.setup()
print("setup equal:", np.array_equal(drv.get_level(0), orc.array(0)))
# relax only
drv.f_relax(0, 0, 256); orc.f_relax(0, 0, 256)
d = np.abs(drv.get_level(0) - orc.array(0)).max(axis=1)
print("after f_relax max err", d.max(), "worst rows", np.argsort(d)[-5:])
r_dev = drv.residual(0, 0, npts); r_orc = orc.residual(0, 0, npts)
e = np.abs(r_dev - r_orc).max(axis=1)
print("residual err", e.max(), np.argsort(e)[-5:])
drv2 = T.CycleDriver(app, hier, cfg); drv2.setup(); orc2 = oracle_driver(args, ic=ic); orc2.setup()
drv2.cycle(); orc2.cycle()
u1, u2 = drv2.get_level(0), orc2.array(0)
d = np.abs(u1 - u2).max(axis=1)
print("after cycle max err", d.max(), "worst rows", np.argsort(d)[-8:], "C rows err", d[::16][:20])
r1 = drv2.get_level(1, 3); r2 = orc2.array(1, 'r')
e = np.abs(r1 - r2).max(axis=1)
print("coarse r err", e.max(), np.argsort(e)[-8:])
bad = np.nonzero(d[::16] > 1e-12)[0]
print("bad C points:", bad.tolist()[:40])
