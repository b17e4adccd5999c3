#!/bin/bash
# A/B of several environment settings on one box: tools/ab_iter.py under each
# argument ("-" = defaults; "A=1,B=2" sets several), alternated twice.
set -u
for r in 1 2; do
  for e in "$@"; do
    if [ "$e" = "-" ]; then timeout 300 python tools/ab_iter.py
    else env ${e//,/ } timeout 300 python tools/ab_iter.py | sed "s/^/$e /"; fi
  done
done
