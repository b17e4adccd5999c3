#!/bin/bash
# ncu full capture of one correction F-sweep launch (config 5), base library
# (tools/ab/libatmgrit_base.so) and in-tree build: raw metrics and SASS page as CSV
mkdir -p gpurun_out
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-ttt-full > /dev/null 2>&1
for v in base new; do
  if [ $v = base ]; then export ATM_LIB=$PWD/tools/ab/libatmgrit_base.so; else unset ATM_LIB; fi
  ncu --set full --clock-control none --import-source on -k regex:heat_sweep -s 3 -c 1 -o /tmp/prof_corr_$v \
      python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-ttt-full > gpurun_out/ncu_corr_$v.log 2>&1; echo "$v rc=$?"
  ncu -i /tmp/prof_corr_$v.ncu-rep --page raw --csv > gpurun_out/corr_raw_$v.csv 2>/dev/null
  ncu -i /tmp/prof_corr_$v.ncu-rep --page source --csv --print-source sass > gpurun_out/corr_sass_$v.csv 2>/dev/null
done
