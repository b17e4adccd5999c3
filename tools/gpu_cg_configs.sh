#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_heat2d.py tests/test_gpu_fullsize.py -k "heat2d or config2" -x -q > gpurun_out/cg_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/cg_tests.log
timeout 300 python tools/configs_probe.py --only 2 --out gpurun_out/cfg2.json > /dev/null 2>&1; echo "cfg2 $(python -c "import json; d=json.load(open('gpurun_out/cfg2.json')); d=d[0] if isinstance(d,list) else d; print(d['ms_per_iteration'], d['inner_iterations'], d['norms'])")"
timeout 900 python tools/configs_probe.py --only 4 --out gpurun_out/cfg4.json > /dev/null 2>&1; echo "cfg4 $(python -c "import json; d=json.load(open('gpurun_out/cfg4.json')); d=d[0] if isinstance(d,list) else d; print(d['ms_per_iteration'], d['inner_iterations'], d['norms'])")"
