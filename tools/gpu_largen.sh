#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -rf -k "phi_matches_oracle or past_4096" > gpurun_out/parity.log 2>&1; echo "parity rc=$?"; grep -E "passed|failed|FAILED|^E " gpurun_out/parity.log | head -30
