#!/bin/bash
# A/B on one box: config-5 iteration (tools/ab_iter.py) and the single-chain
# Phi latency (tools/seqphi_probe.py), baseline library tools/ab/libatmgrit_base.so
# against the in-tree build, alternated twice.
set -u
mkdir -p gpurun_out
for r in 1 2; do
  ATM_LIB=$PWD/tools/ab/libatmgrit_base.so timeout 300 python tools/ab_iter.py
  timeout 300 python tools/ab_iter.py
done
ATM_LIB=$PWD/tools/ab/libatmgrit_base.so python tools/seqphi_probe.py 16385
python tools/seqphi_probe.py 16385
