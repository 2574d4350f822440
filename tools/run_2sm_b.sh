#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_nn.py -q --timeout 120 > gpurun_out/tc2b_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tc2b_tests.log
timeout 600 python bench.py --config mlp_wide --steps 20 > gpurun_out/mlpw2_n1.json 2> gpurun_out/mlpw2_n1.err
NCU=/usr/local/cuda/bin/ncu
$NCU --set full --clock-control none --import-source on -k regex:gemm_tc2_kernel -s 2 -c 1 -o gpurun_out/ncu_gemm2_wide -f python tools/gemm_one.py 4 > gpurun_out/ncu_gemm2.log 2>&1
python tools/ncu_summary.py gemm_tc2_wide_fwd:gpurun_out/ncu_gemm2_wide.ncu-rep > gpurun_out/r02_ncu_gemm2.md 2>&1
rm -f gpurun_out/*.ncu-rep
