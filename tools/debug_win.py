import sys, os, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2107_09596_b200 as T
from helpers import device_objects, oracle_driver
from oracle import oracle as O
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4095
npts, k = 4097, 8
ic = O.random_state(7, n)
args = dict(problem="heat1d", n=n, tf=1.0, n_points=npts, m=16, k=k, manufactured=0, guess="random", seed=20, tol=1e-10, max_iters=2)
os.environ["ATM_DEBUG_DUMP"] = "/tmp/dbg"
app, hier, cfg = device_objects(args, ic=ic)
drv = T.CycleDriver(app, hier, cfg); drv.setup(); drv.cycle()
P = (n + 15) // 16 * 16
rb = np.fromfile("/tmp/dbg_r_before").reshape(-1, P)[:, :n]
ra = np.fromfile("/tmp/dbg_r_after").reshape(-1, P)[:, :n]
ub = np.fromfile("/tmp/dbg_u_before").reshape(-1, P)[:, :n]
ua = np.fromfile("/tmp/dbg_u_after").reshape(-1, P)[:, :n]
print("r changed by window kernel:", np.abs(ra - rb).max())
orc = oracle_driver(args, ic=ic)
nc = rb.shape[0]
bad = []
for p in range(nc):
    lo = max(0, p - k + 1)
    e = orc.window_linear(1, lo, rb[lo:p + 1])
    want = ub[16 * p] + e
    err = np.abs(ua[16 * p] - want).max()
    if err > 1e-12:
        bad.append((p, float(err)))
fmask = np.ones(ua.shape[0], bool); fmask[::16] = False
print("F rows changed:", np.abs(ua[fmask] - ub[fmask]).max())
print("bad windows:", bad[:30])
