#!/bin/bash
# ncu evidence (one GPU): tcgen05 GEMM full set; launch lists of the MLP and lab benches
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
python tools/gemm_one.py 3 > gpurun_out/gemm_one.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 2 -c 1 -o gpurun_out/ncu_gemm_wide -f python tools/gemm_one.py 4 > gpurun_out/ncu_gemm.log 2>&1
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_mlp.csv python bench.py --config mlp --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_mlp.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:optimizer_kernel -s 20 -c 1 -o gpurun_out/ncu_opt_wide -f python bench.py --config mlp_wide --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_opt.log 2>&1
python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err
