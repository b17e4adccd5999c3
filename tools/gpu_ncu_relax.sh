#!/bin/bash
# ncu full capture of one relax F-sweep launch (config 5): raw metrics (every
# warp-stall reason) and the SASS source page, as CSV
mkdir -p gpurun_out
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-ttt-full > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:heat_sweep -s 2 -c 1 -o /tmp/prof_relax \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-ttt-full > gpurun_out/ncu_relax.log 2>&1; echo "relax rc=$?"
ncu -i /tmp/prof_relax.ncu-rep --page raw --csv > gpurun_out/relax_raw.csv 2>/dev/null; echo "raw rc=$?"
ncu -i /tmp/prof_relax.ncu-rep --page source --csv --print-source sass > gpurun_out/relax_sass.csv 2>/dev/null; echo "csv rc=$?"
ls -la gpurun_out/relax_*.csv
