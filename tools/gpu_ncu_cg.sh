#!/bin/bash
# ncu --set full of one strip-CG window launch (config 2)
mkdir -p gpurun_out
export ATM_CG_STRIP_E=${ATM_CG_STRIP_E:-16}
python tools/configs_probe.py --only 2 --out gpurun_out/ncu_plain.json > /dev/null 2>&1; echo "plain rc=$?"
ncu --set full --clock-control none --import-source on -k regex:cg_window_kernel -s 1 -c 1 -o gpurun_out/prof_cg2_win \
  python tools/configs_probe.py --only 2 --out gpurun_out/ncu_run2.json > gpurun_out/ncu_cg2w.log 2>&1; echo "ncu win rc=$?"
