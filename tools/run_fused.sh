#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_nn.py -q --timeout 300 > gpurun_out/fused_tests.log 2>&1; echo "rc=$?" >> gpurun_out/fused_tests.log
timeout 600 python bench.py --config mlp > gpurun_out/mlpf_n1.json 2> gpurun_out/mlpf_n1.err
timeout 600 python bench.py --config mlp_wide --steps 20 > gpurun_out/mlpwf_n1.json 2> gpurun_out/mlpwf_n1.err
timeout 600 python bench.py --config mlp --dtype f32 --no-e2e > gpurun_out/mlpf32_n1.json 2> gpurun_out/mlpf32_n1.err
