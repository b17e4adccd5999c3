#!/bin/bash
# NOTE: compute-sanitizer is closed on this pool (runs under it left GPUs
# needing a reset); kept for boxes where it is allowed.
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_cases.py
# (one process per case and tool, each bounded), logs to gpurun_out/sanitize/
mkdir -p gpurun_out/sanitize
cases="${@:-heat_two_level heat_l32_fcf heat_fas allen_cahn heat2d heat2d_big gray_scott}"
for tool in memcheck synccheck racecheck; do
  for c in $cases; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py $c \
      > gpurun_out/sanitize/${tool}_${c}.log 2>&1
    echo "$tool $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize/${tool}_${c}.log | tail -1)"
  done
done
