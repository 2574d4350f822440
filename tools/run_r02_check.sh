#!/bin/bash
# Round-2 check: GPU tests, N=1 bench (resnet18, parity pass), GPT-2-scale bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,memory.used --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "rc=$?" >> gpurun_out/bench_n1.err
timeout 900 python bench.py --config gpt2 --steps 8 --warmup 3 --e2e-steps 2 > gpurun_out/bench_gpt2.json 2> gpurun_out/bench_gpt2.err; echo "rc=$?" >> gpurun_out/bench_gpt2.err
