#!/bin/bash
# A/B of an environment switch on one box: tools/ab_iter.py with "$1" set
# (e.g. ATM_RELAX1=0) against the default, alternated twice.
set -u
for r in 1 2; do
  env $1 timeout 300 python tools/ab_iter.py
  timeout 300 python tools/ab_iter.py
done
