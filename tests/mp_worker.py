"""One rank of a multi-process AT-MGRIT solve through the engine's
one-shard-per-process path (atm_runtime.world_size > 1), with the
host-mediated NCCL stand-in (tests/mocknccl) so several processes can share
the single GPU.  Spawned by tests/test_gpu_multiproc.py:

    ATM_NCCL_LIB=... python tests/mp_worker.py CASE RANK WORLD IDFILE OUT.npz

MP_DIE_RANK=r makes rank r exit right after setup (a crashed peer); the
other ranks record the error their solve raised (status, message, seconds).
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import ctypes as C  # noqa: E402

import paper_2107_09596_b200 as T  # noqa: E402
from mp_cases import build_case  # noqa: E402


def main():
    case, rank, world, idfile, out = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5]
    if rank == 0:
        buf = (C.c_char * 128)()
        assert T.lib().atm_nccl_unique_id(buf) == 0
        with open(idfile + ".tmp", "wb") as f:
            f.write(bytes(buf))
        os.rename(idfile + ".tmp", idfile)
    t0 = time.time()
    while not os.path.exists(idfile):
        if time.time() - t0 > 120:
            raise SystemExit("no nccl id")
        time.sleep(0.01)
    nid = open(idfile, "rb").read()
    app, hier, cfg = build_case(case)
    drv = T.CycleDriver(app, hier, cfg, world_size=world, rank=rank, nccl_id=nid,
                        timeout_ms=int(os.environ.get("MP_TIMEOUT_MS", "0")))
    if os.environ.get("MP_DIE_RANK") is not None:
        drv.setup()
        if rank == int(os.environ["MP_DIE_RANK"]):
            os._exit(0)  # a peer that dies without a word
        t = time.time()
        try:
            drv.drive()
            err = dict(error=None)
        except T.TempoError as e:
            err = dict(error=type(e).__name__, what=str(e))
        err["seconds"] = time.time() - t
        with open(out + ".json", "w") as f:
            json.dump(err, f)
        os._exit(0)
    rep = drv.drive()
    rr = T.rank_ranges(hier, world, rank)
    lo, hi = rr["lo"][0], rr["hi"][0]
    u = drv.get_level(0, first=lo, count=hi - lo + 1)
    np.savez(out, norms=np.array(rep.residual_norms), iterations=rep.iterations, lo=lo, hi=hi, u=u)


if __name__ == "__main__":
    main()
