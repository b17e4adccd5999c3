#!/bin/bash
# Round profiling recipe (B200_PROFILING.md): plain bench, launch list, full
# captures of the two level-0 sweeps (relax, correction), the window kernel
# and the strip CG (config 2 cluster mode, config 4 group mode).
#   CONFIG5_SWEEP=1 also runs the full-size m x k sweep (long)
set -u
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-ttt-full > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-ttt-full > gpurun_out/ncu_list.log 2>&1; echo "list rc=$?"
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-ttt-full > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:heat_sweep -s 2 -c 2 -o gpurun_out/prof_sweep \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-ttt-full > gpurun_out/ncu_sweep.log 2>&1; echo "sweep rc=$?"
ncu --set full --clock-control none --import-source on -k regex:heat_window_linear -s 1 -c 1 -o gpurun_out/prof_win \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-ttt-full > gpurun_out/ncu_win.log 2>&1; echo "win rc=$?"
bash tools/gpu_ncu_cg.sh
if [ "${CONFIG5_SWEEP:-0}" = 1 ]; then
  python tools/config5_sweep.py gpurun_out/config5_sweep.json > gpurun_out/config5_sweep.log 2>&1; echo "config5 sweep rc=$?"
fi
python tools/seqphi_probe.py > gpurun_out/seqphi.txt 2>&1; echo "seqphi rc=$?"
# summaries on the box (the .ncu-rep files exceed gpurun_out's 64 MiB cap)
python tools/ncu_summary.py gpurun_out/ncu_sweep_summary.json sweep=gpurun_out/prof_sweep.ncu-rep \
    win=gpurun_out/prof_win.ncu-rep --alg=8587837440 --dominant=sweep#1 > /dev/null 2>&1; echo "summary rc=$?"
python tools/ncu_summary.py gpurun_out/ncu_cg_summary.json cg2=gpurun_out/prof_cg2_win.ncu-rep \
    cg4=gpurun_out/prof_cg4_win.ncu-rep > /dev/null 2>&1; echo "cg summary rc=$?"
rm -f gpurun_out/*.ncu-rep
