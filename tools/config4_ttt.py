"""BASELINE config 4 at full size on one B200: 2D heat 511^2, N_t = 65536 over
[0, 4], four-level FAS V-cycle m = (8, 8, 8), k = 2, CG Phi (rtol 1e-12),
Fourier u0, random guess (seed 20), tol 1e-10.  Level 0 uses C-point storage
(the full level-0 array, 137 GB, does not fit one GPU with the other levels).
One JSON line per cycle (flushed) so a cut-off run still reports progress.

  python tools/config4_ttt.py out.jsonl [max_cycles] [reuse]

`reuse` adds the relax-reuse opt-in (the level-0 opening F-sweep of every
cycle after the first is skipped; bitwise the same cycles)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2107_09596_b200 as T  # noqa: E402

out = open(sys.argv[1], "w")
max_cycles = int(sys.argv[2]) if len(sys.argv) > 2 else 80
reuse = len(sys.argv) > 3 and sys.argv[3] == "reuse"
app = T.Heat2D(511, folded=True, source=None, cg_rtol=1e-12, initial_condition=T.fourier_ic(511))
hier = T.build_hierarchy(T.TimeGrid.make(0.0, 4.0, 65537), [8, 8, 8], 2)
cfg = T.SolverConfig(mode=T.CycleMode.VCycle, relaxation=T.Relaxation.F, max_iters=max_cycles, tol=1e-10,
                     initial_guess=T.InitialGuess.Random, seed=20)
t0 = time.perf_counter()
drv = T.CycleDriver(app, hier, cfg, cpoint_storage=True, reuse_relax=reuse)
drv.setup()
out.write(json.dumps({"setup_s": time.perf_counter() - t0, "relax_reuse": reuse}) + "\n")
out.flush()
for it in range(1, max_cycles + 1):
    v = float(drv.iterate(1)[0])
    rec = {"cycle": it, "norm": v, "wall_s": time.perf_counter() - t0,
           "inner_cg_iterations": drv.inner_iterations()}
    out.write(json.dumps(rec) + "\n")
    out.flush()
    if v <= 1e-10:
        break
drv.close()
