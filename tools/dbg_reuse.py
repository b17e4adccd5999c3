import sys, time
sys.path.insert(0, '/root/repo')
import paper_2107_09596_b200 as T
n, npts = 4095, 2 ** 14 + 1
app = T.Heat1D(n, manufactured_forcing=False, initial_condition=T.random_state(7, n))
hier = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, npts), [16], 8)
cfg = T.SolverConfig(mode=T.CycleMode.TwoLevel, relaxation=T.Relaxation.F, tol=1e-10, max_iters=400,
                     initial_guess=T.InitialGuess.Random, seed=20)
for rep in range(3):
    for reuse in (False, True):
        drv = T.CycleDriver(app, hier, cfg, reuse_relax=reuse)
        drv.setup()
        t0 = time.perf_counter()
        r = drv.drive()
        dt = time.perf_counter() - t0
        print('reuse', reuse, 'iters', r.iterations, 'drive %.4f s' % dt, 'per-iter %.3f ms' % (dt / r.iterations * 1e3))
        drv.close()
