set -x
K="--kernel-name-base demangled --set full --clock-control none --import-source on -c 1"
ncu $K -k 'regex:int.64, .bool.0, .bool.0, __nv_bfloat16, .int.1' -o gpurun_out/cnn_fwd64 python tools/cnn_step_profile.py 8 128 1 > /dev/null 2>&1
ncu $K -k 'regex:int.64, .bool.0, .bool.1, __nv_bfloat16, .int.3' -o gpurun_out/cnn_dgrad64 python tools/cnn_step_profile.py 8 128 1 > /dev/null 2>&1
ncu $K -k 'regex:int.256, .bool.1, .bool.1, float, .int.2' -o gpurun_out/cnn_wgrad python tools/cnn_step_profile.py 8 128 1 > /dev/null 2>&1
ncu $K -k 'regex:int.256, .bool.0, .bool.0, __nv_bfloat16, .int.1' -o gpurun_out/cnn_fwd256 python tools/cnn_step_profile.py 8 128 1 > /dev/null 2>&1
python tools/ncu_summary.py fwd64:gpurun_out/cnn_fwd64.ncu-rep dgrad64:gpurun_out/cnn_dgrad64.ncu-rep wgrad:gpurun_out/cnn_wgrad.ncu-rep fwd256:gpurun_out/cnn_fwd256.ncu-rep > gpurun_out/cnn_ncu.md
rm -f gpurun_out/*.ncu-rep
