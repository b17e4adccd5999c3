#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_heat2d.py -x -q > gpurun_out/cg4_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/cg4_tests.log
for lvl in 0 3; do timeout 600 python tools/cg_probe.py 511 8 $lvl 4 2>&1 | tail -1; done
for v in "ATM_CG_GROUP=1" "ATM_CG_GROUP=0"; do
  env $v timeout 900 python tools/configs_probe.py --only 4 --out gpurun_out/cfg4.json > /dev/null 2>&1; echo "$v $(python -c "import json; d=json.load(open('gpurun_out/cfg4.json')); d=d[0] if isinstance(d,list) else d; print(d['ms_per_iteration'], d['inner_iterations'], d['norms'])")"
done
