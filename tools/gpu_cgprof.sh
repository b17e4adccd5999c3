#!/bin/bash
# per-phase cycle counts of the strip CG loop (clock64 probe; library built
# with -DATM_CG_PROF into tools/prof/libatmgrit_prof.so)
for lvl in 0 3; do ATM_LIB=$PWD/tools/prof/libatmgrit_prof.so timeout 600 python tools/cg_probe.py 511 8 $lvl 4 2>&1 | grep -E "cgprof|^\{" | sort | uniq -c | sort -rn | head -8; done
ATM_LIB=$PWD/tools/prof/libatmgrit_prof.so timeout 600 python tools/cg_probe.py 127 64 0 2 2>&1 | grep -E "cgprof|^\{" | head -6
