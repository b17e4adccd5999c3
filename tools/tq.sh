#!/bin/bash
# quick timing line: value ms_per_step frac sweep_correct coarse
python bench.py --steps 6 --warmup 2 --no-e2e --no-cpu "$@" 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read());p=d['phase_ms_per_step'];print('%.3e ms=%.3f frac=%.3f sweep=%.3f coarse=%.3f'%(d['value'],d['ms_per_step'],d['roofline']['frac'],p['sweep_correct'],p['coarse']))"
