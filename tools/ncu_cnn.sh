# ncu --set full of the conv stack's main kernels (one launch each) -> gpurun_out/cnn_ncu.md
K="--kernel-name-base demangled --set full --clock-control none --import-source on -c 1"
ncu $K -k 'regex:conv64_kernel<.int.1>' -o gpurun_out/cnn_c64f python tools/cnn_step_profile.py 8 128 1 > /dev/null 2>&1
ncu $K -k 'regex:conv64_kernel<.int.3>' -o gpurun_out/cnn_c64d python tools/cnn_step_profile.py 8 128 1 > /dev/null 2>&1
ncu $K -k 'regex:int.256, .bool.1, .bool.1, float, .int.2' -o gpurun_out/cnn_wgrad python tools/cnn_step_profile.py 8 128 1 > /dev/null 2>&1
ncu $K -k 'regex:int.64, .bool.1, .bool.1, float, .int.4' -o gpurun_out/cnn_wgradT python tools/cnn_step_profile.py 8 128 1 > /dev/null 2>&1
ncu $K -k 'regex:int.256, .bool.0, .bool.0, __nv_bfloat16, .int.1, .bool.1' -o gpurun_out/cnn_fwd256 python tools/cnn_step_profile.py 8 128 1 > /dev/null 2>&1
python tools/ncu_summary.py conv64_fwd:gpurun_out/cnn_c64f.ncu-rep conv64_dgrad:gpurun_out/cnn_c64d.ncu-rep \
  wgrad_s1to3:gpurun_out/cnn_wgrad.ncu-rep wgradT_s0:gpurun_out/cnn_wgradT.ncu-rep fwd_bn256:gpurun_out/cnn_fwd256.ncu-rep \
  > gpurun_out/cnn_ncu.md 2>&1
rm -f gpurun_out/*.ncu-rep
