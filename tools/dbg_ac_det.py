import sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2107_09596_b200 as T
n = 4096
app = T.AllenCahn(n, 0.02, 1.0, 1e-12, 30, initial_condition=T.allen_cahn_ic(n))
hier = T.build_hierarchy(T.TimeGrid.make(0.0, 8.0, 16385), [8, 8], 4)
sc = T.SolverConfig(mode=T.CycleMode.VCycle, relaxation=T.Relaxation.F, max_iters=100, tol=1e-10,
                    initial_guess=T.InitialGuess.Random, seed=20)
xs = np.stack([T.random_state(100 + j, n) for j in range(64)])
drv = T.CycleDriver(app, hier, sc)
for level in (0, 1, 2):
    ref = drv.apply_phi(level, 1, xs)
    bad = 0
    for rep in range(5):
        got = drv.apply_phi(level, 1, xs)
        bad += int(not np.array_equal(got, ref))
    print('apply level', level, 'mismatching repeats', bad, flush=True)
res = []
for rep in range(3):
    d = T.CycleDriver(app, hier, sc)
    d.setup()
    res.append(d.iterate(2))
    print('cycle norms', res[-1], flush=True)
# sweep determinism: F-relax twice from the same state
d = T.CycleDriver(app, hier, sc); d.setup(); u0 = d.get_level(0)
d.f_relax(0, 0, 2048); a = d.get_level(0)
d.set_level(0, u0); d.f_relax(0, 0, 2048); b = d.get_level(0)
print('f_relax bitwise', np.array_equal(a, b), np.max(np.abs(a - b)))
