#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python bench.py --config llama_mlp --steps 5 --warmup 3 --e2e-steps 2 > gpurun_out/llama_n1.json 2> gpurun_out/llama_n1.err
timeout 1500 python tools/run_nn_modes.py --llama > gpurun_out/nn_modes2.json 2> gpurun_out/nn_modes2.err
