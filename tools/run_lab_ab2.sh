#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export DSX_FLAG_TIMEOUT_S=120
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multigpu.py tests/test_gpu_config1.py -q --timeout 600 -x > gpurun_out/lab_tests2.log 2>&1; echo "rc=$?" >> gpurun_out/lab_tests2.log
unset DSX_FLAG_TIMEOUT_S
timeout 600 python bench.py --workers 2 --no-e2e --no-cpu-baseline > gpurun_out/k2_n1.json 2> gpurun_out/k2_n1.err
for n in 2 4; do timeout 900 python bench.py --gpus $n > gpurun_out/lab_n$n.json 2> gpurun_out/lab_n$n.err; done
