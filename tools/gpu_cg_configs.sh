#!/bin/bash
# config-2 / config-4 iteration time under CG geometry variants (VARIANTS="A=1 B=2,C=3"; "-" = defaults)
mkdir -p gpurun_out
for v in ${VARIANTS:--}; do
  e=""; [ "$v" != "-" ] && e="${v//,/ }"
  env $e timeout 300 python tools/configs_probe.py --only ${CONFIGS:-2} --out gpurun_out/cfgv.json > /dev/null 2>&1
  echo "$v $(python -c "import json; [print(d['config'][:8], round(d['ms_per_iteration'],2), d['inner_iterations']) for d in json.load(open('gpurun_out/cfgv.json'))]")"
done
