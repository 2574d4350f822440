#!/bin/bash
# 2-GPU evidence: GPU test suites needing 2 GPUs, MLP + lab benches at N=2
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multigpu_nn.py tests/test_gpu_multigpu.py -q > gpurun_out/multi2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/multi2_tests.log
timeout 600 python bench.py --config mlp --gpus 2 > gpurun_out/mlp_n2.json 2> gpurun_out/mlp_n2.err; echo "rc=$?" >> gpurun_out/mlp_n2.err
timeout 600 python bench.py --config mlp > gpurun_out/mlp_n1.json 2> gpurun_out/mlp_n1.err; echo "rc=$?" >> gpurun_out/mlp_n1.err
timeout 900 python bench.py --gpus 2 > gpurun_out/lab_n2.json 2> gpurun_out/lab_n2.err; echo "rc=$?" >> gpurun_out/lab_n2.err
