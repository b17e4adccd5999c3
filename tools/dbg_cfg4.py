import sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2107_09596_b200 as T
nx, npts, ms = 511, 17, [8]
app = T.Heat2D(nx, folded=False, source=None, cg_rtol=1e-12, initial_condition=T.fourier_ic(nx))
hier = T.build_hierarchy(T.TimeGrid.make(0.0, 0.01, npts), ms, 2)
sc = T.SolverConfig(mode=T.CycleMode.TwoLevel, relaxation=T.Relaxation.F, max_iters=3, tol=1e-10,
                    initial_guess=T.InitialGuess.Random, seed=20)
drv = T.CycleDriver(app, hier, sc)
drv.setup(); print('setup ok', flush=True)
for name, f in [('resid1', lambda: drv.residual(0, 5, 1)), ('resid_all', lambda: drv.residual(0, 0, npts)),
                ('norm', lambda: drv.residual_norm()), ('apply1', lambda: drv.apply_phi(1, 1, np.ones((1, nx*nx)))),
                ('cycle', lambda: drv.iterate(1))]:
    try:
        out = f(); print(name, 'ok', np.ravel(out)[:2], flush=True)
    except Exception as e:
        print(name, 'FAIL', e, flush=True); break
