"""The engine's one-shard-per-process path (atm_runtime.world_size > 1: NCCL
halo / window payload / norm all-reduce / nested chain) run as 2-3 processes
on the single GPU, with the host-mediated NCCL stand-in tests/mocknccl (real
NCCL needs one GPU per rank).  Histories must be bitwise those of the
single-process solve (the reference's contract across rank counts,
test_runtime.cpp:194-228) and the assembled level-0 state bitwise equal."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

import numpy as np
import pytest

import paper_2107_09596_b200 as T
from mp_cases import build_case

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
MOCK = os.path.join(HERE, "mocknccl", "libmocknccl.so")


def _mock_lib():
    subprocess.check_call(["make", "-s", "-C", os.path.join(HERE, "mocknccl")])
    return MOCK


@pytest.mark.parametrize("case,world", [("two_level", 2), ("two_level", 3), ("fas_vcycle", 2),
                                        ("nested_fcf", 3), ("global_coarse", 2), ("heat2d_strip", 2),
                                        ("heat2d_group", 2), ("allen_cahn", 2),
                                        ("heat1d_cluster_rows", 2), ("gray_scott", 2)])
def test_multiprocess_solve_bitwise_equals_single_process(case, world):
    lib = _mock_lib()
    app, hier, cfg = build_case(case)
    ref = T.solve(app, hier, cfg)
    tmp = tempfile.mkdtemp(prefix="mp_")
    try:
        idfile = os.path.join(tmp, "nccl.id")
        env = dict(os.environ, ATM_NCCL_LIB=lib)
        procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "mp_worker.py"), case, str(r),
                                   str(world), idfile, os.path.join(tmp, f"r{r}.npz")], env=env)
                 for r in range(world)]
        for p in procs:
            assert p.wait(timeout=600) == 0
        u = np.zeros_like(ref.state)
        for r in range(world):
            d = np.load(os.path.join(tmp, f"r{r}.npz"))
            assert int(d["iterations"]) == ref.report.iterations
            assert np.array_equal(d["norms"], np.array(ref.report.residual_norms)), (r, d["norms"])
            u[int(d["lo"]):int(d["hi"]) + 1] = d["u"]
        assert np.array_equal(u, ref.state)
    finally:
        _cleanup(tmp)


def _cleanup(tmp):
    shutil.rmtree(tmp, ignore_errors=True)
    for f in os.listdir("/dev/shm"):
        if f.startswith("mocknccl_"):
            shutil.rmtree(os.path.join("/dev/shm", f), ignore_errors=True)


def test_dead_rank_surfaces_as_runtime_fault_within_the_timeout():
    # parallel.cpp:365-383 / transport.cpp:29-61: a rank that dies must not
    # hang the others -- they fail with RuntimeFault once the exchange times out
    lib = _mock_lib()
    tmp = tempfile.mkdtemp(prefix="mp_")
    try:
        idfile = os.path.join(tmp, "nccl.id")
        env = dict(os.environ, ATM_NCCL_LIB=lib, MP_DIE_RANK="1", MOCKNCCL_TIMEOUT_MS="3000",
                   MP_TIMEOUT_MS="3000")
        procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "mp_worker.py"), "two_level", str(r),
                                   "2", idfile, os.path.join(tmp, f"r{r}.npz")], env=env)
                 for r in range(2)]
        for p in procs:
            assert p.wait(timeout=120) == 0
        import json
        err = json.load(open(os.path.join(tmp, "r0.npz.json")))
        assert err["error"] == "RuntimeFault", err
        assert "timed out" in err["what"], err
        assert err["seconds"] < 30, err
    finally:
        _cleanup(tmp)


def test_bench_spawns_its_own_ranks():
    # bench.py --gpus 2 without a launcher re-launches itself through
    # torch.distributed.run (every rank on device 0 with BENCH_SHARE_DEVICE
    # and the host-mediated stand-in): the line reports the 2 ranks
    lib = _mock_lib()
    env = dict(os.environ, ATM_NCCL_LIB=lib, BENCH_SHARE_DEVICE="1")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(os.path.dirname(HERE), "bench.py"), "--gpus", "2",
                          "--steps", "3", "--warmup", "1", "--n-points", "4097", "--no-e2e", "--no-cpu",
                          "--no-ttt-full"], env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    import json
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0
    # and a launcher whose world size disagrees with --gpus is refused
    bad = subprocess.run([sys.executable, os.path.join(os.path.dirname(HERE), "bench.py"), "--gpus", "2"],
                         env=dict(env, WORLD_SIZE="1"), capture_output=True, text=True, timeout=120)
    assert bad.returncode != 0
