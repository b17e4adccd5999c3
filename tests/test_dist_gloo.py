"""CPU multi-process: the sharded (time-parallel) schedule over gloo with
world_size 2 reproduces the sequential solve bitwise -- the reference's
determinism contract (tests/test_runtime.cpp:194-228)."""
import json
import os
import socket
import subprocess
import sys
import tempfile

import numpy as np
import pytest

from helpers import oracle_driver

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_gloo_history_bitwise_equals_sequential(world):
    sys.path.insert(0, HERE)
    from dist_worker import CASE
    out = tempfile.mktemp(suffix=".json")
    port = str(_free_port())
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "dist_worker.py"), str(r),
                               str(world), port, out], env=env)
             for r in range(world)]
    for p in procs:
        assert p.wait(timeout=300) == 0
    got = json.load(open(out))
    seq = oracle_driver(CASE)
    ref = seq.drive()
    assert got["history"] == ref["history"].tolist()
    assert np.array_equal(np.array(got["u"]), seq.array(0))
