#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export DSX_FLAG_TIMEOUT_S=120
timeout 900 python -m pytest tests/test_gpu_nn.py tests/test_gpu_multigpu_nn.py -q --timeout 300 > gpurun_out/graph_tests.log 2>&1; echo "rc=$?" >> gpurun_out/graph_tests.log
for n in 1 2; do
  timeout 600 python bench.py --config mlp --gpus $n > gpurun_out/mlpg_n$n.json 2> gpurun_out/mlpg_n$n.err
done
timeout 600 python bench.py --config mlp --no-graphs --no-cpu-baseline --no-e2e > gpurun_out/mlp_nog_n1.json 2> gpurun_out/mlp_nog_n1.err
