#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python bench.py --config mlp > gpurun_out/mlp_n1.json 2> gpurun_out/mlp_n1.err; echo "rc=$?" >> gpurun_out/mlp_n1.err
timeout 600 python bench.py --config mlp --dtype f32 --no-e2e > gpurun_out/mlp_f32_n1.json 2> gpurun_out/mlp_f32_n1.err; echo "rc=$?" >> gpurun_out/mlp_f32_n1.err
timeout 600 python bench.py --config mlp_wide --steps 20 > gpurun_out/mlpw_n1.json 2> gpurun_out/mlpw_n1.err; echo "rc=$?" >> gpurun_out/mlpw_n1.err
