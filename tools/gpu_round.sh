#!/bin/bash
# round-2 first GPU call: box info, FP64 peak, smoke, -m gpu suite, bench
mkdir -p gpurun_out
{ nproc; free -g; lscpu | grep -E "Model name|Socket|Core|Thread|NUMA node\(s\)"; nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv; } > gpurun_out/box.txt 2>&1
./tools/ubench/fp64_peak > gpurun_out/fp64_peak.json 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 3000 python -m pytest tests -m gpu -q -rf --durations=25 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/pytest_gpu.log
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json | head -c 3000
