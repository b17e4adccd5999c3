import sys, time, json
sys.path.insert(0, '/root/repo')
import paper_2107_09596_b200 as T
nx = int(sys.argv[1]) if len(sys.argv) > 1 else 127
app = T.Heat2D(nx, folded=False, source=T.gaussian_source(nx), cg_rtol=1e-12)
hier = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, 4097), [16], 4)
sc = T.SolverConfig(mode=T.CycleMode.TwoLevel, relaxation=T.Relaxation.F, max_iters=100, tol=1e-10,
                    initial_guess=T.InitialGuess.Random, seed=20)
drv = T.CycleDriver(app, hier, sc, trace=True)
drv.setup(); drv.iterate(1)
norms, ms = drv.iterate_timed(2)
print('ms/iter', ms / 2)
print(json.dumps(drv.timings(with_counts=True), indent=0)[:2000])
