#!/bin/bash
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-ttt-full > gpurun_out/qb.json 2> gpurun_out/qb.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/qb.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac']); print(json.dumps(d['roofline_fp64'], indent=1)); print(d['phase_ms_per_step'])"
