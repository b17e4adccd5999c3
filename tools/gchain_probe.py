import sys, os
sys.path.insert(0, os.getcwd())
import paper_2107_09596_b200 as T
N, NPTS, m = 4095, 2**16 + 1, 16
app = T.Heat1D(N, manufactured_forcing=False, initial_condition=T.random_state(7, N))
n_c = (NPTS - 1)//m + 1
hier = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, NPTS), [m], n_c)
cfg = T.SolverConfig(relaxation=T.Relaxation.F, tol=1e-300, max_iters=5, initial_guess=T.InitialGuess.Random, seed=20)
drv = T.CycleDriver(app, hier, cfg, trace=True)
drv.setup(); drv.iterate(1); t0 = drv.timings(); drv.iterate(1); t1 = drv.timings()
print({k: 1e3*(t1[k]-t0.get(k,0)) for k in t1}, "us per coarse step", 1e6*(t1['coarse']-t0['coarse'])/(n_c-1))
