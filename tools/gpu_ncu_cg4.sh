#!/bin/bash
mkdir -p gpurun_out
for lvl in 0 3; do timeout 600 python tools/cg_probe.py 511 8 $lvl 4 2>&1 | tail -1; done
ncu --set full --clock-control none --import-source on -k regex:cg_window_kernel -s 1 -c 1 -o gpurun_out/prof_cg4g \
  python tools/cg_probe.py 511 8 0 4 > gpurun_out/ncu_cg4.log 2>&1; echo "ncu rc=$?"
