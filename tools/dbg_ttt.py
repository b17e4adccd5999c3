import sys, time
sys.path.insert(0, '/root/repo')
import paper_2107_09596_b200 as T
n, npts = 4095, 2 ** 14 + 1
app = T.Heat1D(n, manufactured_forcing=False, initial_condition=T.random_state(7, n))
hier = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, npts), [16], 8)
cfg = T.SolverConfig(mode=T.CycleMode.TwoLevel, relaxation=T.Relaxation.F, tol=1e-10, max_iters=400,
                     initial_guess=T.InitialGuess.Random, seed=20)
for rep in range(2):
    t0 = time.perf_counter()
    drv = T.CycleDriver(app, hier, cfg, trace=True)
    t1 = time.perf_counter()
    drv.setup()
    t2 = time.perf_counter()
    rep_ = drv.drive()
    t3 = time.perf_counter()
    print('create %.4f setup %.4f drive %.4f iters %d per-iter %.3f ms' % (t1-t0, t2-t1, t3-t2, rep_.iterations, (t3-t2)/rep_.iterations*1e3))
    tm = drv.timings(with_counts=True)
    print({k: (round(v[0]*1e3/ rep_.iterations, 4), v[1]) for k, v in tm.items()})
d2 = T.CycleDriver(app, hier, cfg); d2.setup(); d2.iterate(3)
norms, ms = d2.iterate_timed(50)
print('iterate_timed per-iter device ms', ms / 50)
