#!/bin/bash
# Full GPU test suite (on however many GPUs the box has), flag waits capped
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export DSX_FLAG_TIMEOUT_S=120
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/gpu_suite.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_suite.log
