#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_multigpu_nn.py -q -x > gpurun_out/multi_api.log 2>&1; echo "rc=$?" >> gpurun_out/multi_api.log
