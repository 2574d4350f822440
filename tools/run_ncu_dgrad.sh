#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
# step 1's kernels: the 2nd (K,N) dgrad launch = the down layer
$NCU --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"tc2_kernel<.int.256, .bool.0, .bool.1" -s 1 -c 1 -o gpurun_out/ncu_dgrad -f python tools/mlp_step_profile.py 1 > gpurun_out/ncu_dgrad.log 2>&1
$NCU --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"tc2_kernel<.int.256, .bool.0, .bool.0, float" -c 1 -o gpurun_out/ncu_head -f python tools/mlp_step_profile.py 1 >> gpurun_out/ncu_dgrad.log 2>&1
python tools/ncu_summary.py dgrad_down:gpurun_out/ncu_dgrad.ncu-rep head_fwd:gpurun_out/ncu_head.ncu-rep > gpurun_out/r02_ncu_dgrad.md 2>&1
$NCU -i gpurun_out/ncu_dgrad.ncu-rep --page source --csv > gpurun_out/ncu_dgrad_source.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
