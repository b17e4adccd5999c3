#!/bin/bash
# ncu --set full of one CG window launch: config 2 (strip kernel, 4-CTA
# clusters) and config 4 (group mode, 37-CTA cooperative groups)
mkdir -p gpurun_out
python tools/configs_probe.py --only 2 --out gpurun_out/ncu_plain.json > /dev/null 2>&1; echo "plain rc=$?"
ncu --set full --clock-control none --import-source on -k regex:cg_window_kernel -s 1 -c 1 -o gpurun_out/prof_cg2_win \
  python tools/configs_probe.py --only 2 --out gpurun_out/ncu_run2.json > gpurun_out/ncu_cg2w.log 2>&1; echo "ncu cfg2 rc=$?"
python tools/cg_probe.py 511 8 0 4 > /dev/null 2>&1; echo "plain4 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:cg_window_kernel -s 1 -c 1 -o gpurun_out/prof_cg4_win \
  python tools/cg_probe.py 511 8 0 4 > gpurun_out/ncu_cg4w.log 2>&1; echo "ncu cfg4 rc=$?"
