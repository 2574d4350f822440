#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_nn.py -q -x > gpurun_out/nn_tests.log 2>&1; echo "rc=$?" >> gpurun_out/nn_tests.log
timeout 600 python tools/gemm_bench.py > gpurun_out/gemm_bench.jsonl 2> gpurun_out/gemm_bench.err
