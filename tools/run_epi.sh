#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_nn.py -q --timeout 120 > gpurun_out/epi_tests.log 2>&1; echo "rc=$?" >> gpurun_out/epi_tests.log
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_llama_slice2.csv python tools/mlp_step_profile.py 2 > gpurun_out/llama_prof2.log 2>&1
timeout 600 python bench.py --config mlp_wide --steps 20 > gpurun_out/mlpw3_n1.json 2> gpurun_out/mlpw3_n1.err
timeout 600 python bench.py --config mlp > gpurun_out/mlp3_n1.json 2> gpurun_out/mlp3_n1.err
