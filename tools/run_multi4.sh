#!/bin/bash
# 4-GPU evidence: the whole GPU suite (incl. 4-rank tests), lab + MLP benches at N=1,2,4
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export DSX_FLAG_TIMEOUT_S=120
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/gpu_suite4.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_suite4.log
unset DSX_FLAG_TIMEOUT_S
for n in 1 2 4; do
  timeout 900 python bench.py --gpus $n > gpurun_out/lab_n$n.json 2> gpurun_out/lab_n$n.err
  timeout 900 python bench.py --config mlp --gpus $n > gpurun_out/mlp_n$n.json 2> gpurun_out/mlp_n$n.err
done
timeout 900 python bench.py --config mlp_wide --steps 20 > gpurun_out/mlpw_n1.json 2> gpurun_out/mlpw_n1.err
timeout 900 python bench.py --config mlp_wide --steps 20 --gpus 4 --no-cpu-baseline > gpurun_out/mlpw_n4.json 2> gpurun_out/mlpw_n4.err
