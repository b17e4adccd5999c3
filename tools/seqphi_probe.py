"""Latency of one Phi on the critical path: a single interval of N_t - 1
steps (m = N_t, one CTA walks the whole chain), so each Phi waits for the
previous one.  Prints device ms and microseconds per Phi of the relax and
correction sweeps (CUDA events).  usage: python tools/seqphi_probe.py [n_points ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_09596_b200 as T  # noqa: E402

N = 4095
for npts in [int(a) for a in sys.argv[1:]] or [2 ** 14 + 1, 2 ** 16 + 1]:
    app = T.Heat1D(N, manufactured_forcing=False, initial_condition=T.random_state(7, N))
    hier = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, npts), [npts - 1], 2)
    cfg = T.SolverConfig(mode=T.CycleMode.TwoLevel, relaxation=T.Relaxation.F, tol=1e-300, max_iters=3,
                         initial_guess=T.InitialGuess.Random, seed=20)
    drv = T.CycleDriver(app, hier, cfg, trace=True)
    drv.setup()
    drv.iterate(1)
    t0 = drv.timings()
    norms, ms = drv.iterate_timed(1)
    t1 = drv.timings()
    d = {k: 1e3 * (t1[k] - t0.get(k, 0.0)) for k in t1}
    nphi = npts - 2
    print(f"n_points {npts}: iteration {ms:.3f} ms; relax sweep {1e3 * d['sweep_relax'] / nphi:.3f} us/Phi, "
          f"correction sweep {1e3 * d['sweep_correct'] / nphi:.3f} us/Phi")
    drv.close()
