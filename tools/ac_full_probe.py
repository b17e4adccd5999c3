"""Config 3 at full size on the device: cycle by cycle until the tolerance or
a Newton failure, for the random guess (seed 20) and the constant (IC) guess.

  python tools/ac_full_probe.py [newton_cap ...]   (default 30)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2107_09596_b200 as T  # noqa: E402

caps = [int(a) for a in sys.argv[1:]] or [30]
for cap, guess in [(c, g) for c in caps for g in (T.InitialGuess.Random, T.InitialGuess.Constant)]:
    app = T.AllenCahn(4096, 0.02, 1.0, float(os.environ.get("NEWTON_TOL", "1e-12")), cap, initial_condition=0.05 * T.random_state(3, 4096))
    hier = T.build_hierarchy(T.TimeGrid.make(0.0, 8.0, 16385), [8, 8], 4)
    cfg = T.SolverConfig(mode=T.CycleMode.VCycle, relaxation=T.Relaxation.F, max_iters=200, tol=1e-10,
                         initial_guess=guess, seed=20)
    d = T.CycleDriver(app, hier, cfg)
    d.setup()
    norms = []
    try:
        for it in range(200):
            v = float(d.iterate(1)[0])
            norms.append(v)
            if v <= 1e-10:
                break
        print("cap", cap, guess, "converged", len(norms), norms[:3], norms[-3:], flush=True)
    except Exception as e:  # noqa: BLE001
        print("cap", cap, guess, "failed at iteration", len(norms) + 1, repr(e), norms[-5:], flush=True)
    d.close()
