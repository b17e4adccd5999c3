mkdir -p gpurun_out
{ nproc; free -g; lscpu | grep -E "Model name|Socket|Core|Thread|NUMA node\(s\)"; nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv; } > gpurun_out/box.txt 2>&1
./tools/ubench/fp64_peak > gpurun_out/fp64_peak.json 2>&1
./tools/ubench/fp64_peak >> gpurun_out/fp64_peak.json 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1; echo "$tool rc=$?"
done
