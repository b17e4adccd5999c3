# full -m gpu suite on the box, log to gpurun_out/
mkdir -p gpurun_out
timeout ${1:-2400} python -m pytest tests -m gpu -q -rf ${2:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu.log
