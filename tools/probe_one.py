"""Run one BASELINE config for a couple of cycles (ncu capture target).
usage: python tools/probe_one.py CONFIG_INDEX"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import configs_probe as P  # noqa: E402

cfg = P.configs()[int(sys.argv[1])]
cfg["iters"] = 1
print(P.run(cfg))
