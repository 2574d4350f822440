#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python tools/mlp_step_profile.py 2 > gpurun_out/llama_prof.log 2>&1
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_llama_slice.csv python tools/mlp_step_profile.py 3 >> gpurun_out/llama_prof.log 2>&1
