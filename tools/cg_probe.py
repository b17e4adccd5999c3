"""2D-heat CG Phi throughput probe (BASELINE config 4 / config 2 shapes):
batched apply_phi of `count` systems on one level, device time via wall
clock around the synchronous call (it includes the H2D/D2H of the batch,
reported separately), inner CG iterations from the device counter ->
DOF x CG-iterations / s.  Run per cluster-size override:

    ATM_DEBUG_OCC=1 ATM_CG_CS=11 python tools/cg_probe.py 511 64 0 4
    args: nx count level m_levels(comma) ; one JSON line per run
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_09596_b200 as T  # noqa: E402


def main():
    nx = int(sys.argv[1]) if len(sys.argv) > 1 else 511
    count = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    level = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    cfgn = int(sys.argv[4]) if len(sys.argv) > 4 else 4
    if cfgn == 4:  # config 4: dt = 4/65536, m = (8, 8, 8)
        hier = T.build_hierarchy(T.TimeGrid.make(0.0, 4.0 * 4096 / 65536, 4097), [8, 8, 8], 2)
        app = T.Heat2D(nx, folded=True, initial_condition=T.fourier_ic(nx))
        mode = T.CycleMode.VCycle
    else:  # config 2: dt = 1/4096, m = 16
        hier = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, 4097), [16], 4)
        app = T.Heat2D(nx, folded=False, source=T.gaussian_source(nx))
        mode = T.CycleMode.TwoLevel
    cfg = T.SolverConfig(mode=mode, tol=1e-10, max_iters=1, initial_guess=T.InitialGuess.Random, seed=20)
    drv = T.CycleDriver(app, hier, cfg)
    x = np.stack([T.random_state(100 + j, nx * nx) for j in range(count)])
    drv.apply_phi(level, 1, x[:2])  # warm-up
    it0 = drv.inner_iterations()
    t = time.perf_counter()
    y = drv.apply_phi(level, 1, x)
    dt = time.perf_counter() - t
    its = drv.inner_iterations() - it0
    print(json.dumps(dict(nx=nx, count=count, level=level, config=cfgn, cs=os.environ.get("ATM_CG_CS"),
                          seconds=dt, cg_iterations=its, cg_per_system=its / count,
                          dof_cg_it_per_s=nx * nx * its / dt, checksum=float(np.sum(y)))), flush=True)


if __name__ == "__main__":
    main()
