#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_nn.py -q --timeout 600 > gpurun_out/nn_tests.log 2>&1; echo "rc=$?" >> gpurun_out/nn_tests.log
