#!/bin/bash
# ncu source-level capture of one coarse-window launch (config 5) -> CSV extract
mkdir -p gpurun_out
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-ttt-full > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:heat_window_linear -s 1 -c 1 -o /tmp/prof_win \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-ttt-full > gpurun_out/ncu_win.log 2>&1; echo "win rc=$?"
ncu -i /tmp/prof_win.ncu-rep --page source --csv --print-source sass > gpurun_out/win_sass.csv 2>/dev/null; echo "csv rc=$?"
ncu -i /tmp/prof_win.ncu-rep --page source --csv --print-source cuda > gpurun_out/win_src.csv 2>/dev/null
ls -la gpurun_out/win_*.csv
