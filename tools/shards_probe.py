"""Config-5 iteration with 1, 2, 4, 8 time shards driven by ONE process on one GPU
(the shard logic of the multi-GPU path; every shard launches its own kernels
on the same stream, so the cost of the split here is launch quantisation, not
communication): ms per iteration and the last norm (bitwise shard-count
independent)."""
import sys, os, json
sys.path.insert(0, os.getcwd())
import paper_2107_09596_b200 as T
n, npts, K = 4095, 2 ** 18 + 1, 10
app = T.Heat1D(n, manufactured_forcing=False, initial_condition=T.random_state(7, n))
hier = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, npts), [16], 8)
cfg = T.SolverConfig(mode=T.CycleMode.TwoLevel, relaxation=T.Relaxation.F, tol=1e-300, max_iters=100,
                     initial_guess=T.InitialGuess.Random, seed=20)
for w in (1, 2, 4, 8):
    drv = T.CycleDriver(app, hier, cfg, workers=w)
    drv.setup(); drv.iterate(2)
    best = 1e9
    for _ in range(3):
        norms, ms = drv.iterate_timed(K); best = min(best, ms / K)
    print(w, round(best, 4), norms[-1]); drv.close()
