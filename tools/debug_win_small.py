import sys, os, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2107_09596_b200 as T
from helpers import device_objects
from oracle import oracle as O
n = 2049
ic = O.random_state(7, n)
args = dict(problem="heat1d", n=n, tf=1.0, n_points=1025, m=16, k=8, manufactured=0, guess="random", seed=20, tol=1e-10, max_iters=2)
app, hier, cfg = device_objects(args, ic=ic)
drv = T.CycleDriver(app, hier, cfg); drv.setup(); drv.cycle()
print("done")
