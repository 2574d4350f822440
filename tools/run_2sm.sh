#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
DSX_GEMM_2SM=1 timeout 400 python -m pytest tests/test_gpu_nn.py -q -x --timeout 120 -k "tc_gemm" > gpurun_out/tc2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tc2_tests.log
DSX_GEMM_2SM=1 timeout 400 python -m pytest tests/test_gpu_nn.py -q -x --timeout 120 -k "mlp" > gpurun_out/tc2_mlp_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tc2_mlp_tests.log
DSX_GEMM_2SM=0 timeout 300 python tools/gemm_bench.py > gpurun_out/gemm_1sm.jsonl 2> gpurun_out/gemm_1sm.err
timeout 300 python tools/gemm_bench.py > gpurun_out/gemm_auto.jsonl 2> gpurun_out/gemm_auto.err
