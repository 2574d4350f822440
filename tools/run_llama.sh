#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python bench.py --config llama_mlp --steps 5 --warmup 3 --e2e-steps 2 > gpurun_out/llama_n1.json 2> gpurun_out/llama_n1.err
nvidia-smi --query-gpu=memory.used --format=csv >> gpurun_out/llama_n1.err
