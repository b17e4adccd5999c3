#!/bin/bash
# strip CG: heat2d parity tests, then config-2 throughput: strip variants vs the smem CG
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_heat2d.py tests/test_gpu_fullsize.py -k "heat2d or config2 or config4" -x -q -rf > gpurun_out/cg_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/cg_tests.log
for v in ${VARIANTS:-"ATM_CG_STRIP=0" "ATM_CG_STRIP_E=16" "ATM_CG_STRIP_E=8"}; do
  f=gpurun_out/cfg2_$(echo $v | tr ' =' '__').json
  env $v timeout 300 python tools/configs_probe.py --only 2 --out $f > /dev/null 2>gpurun_out/cfg2_err.log
  echo "$v: $(python -c "import json,sys; d=json.load(open('$f')); d=d[0] if isinstance(d,list) else d; print(d['ms_per_iteration'], d['inner_iterations'], d['norms'])")"
done
