K="--kernel-name-base demangled --set full --clock-control none --import-source on -c 1"
ncu $K -k 'regex:int.64, .bool.0, .bool.0, __nv_bfloat16, .int.1' -o gpurun_out/cnn_fwd64 python tools/cnn_step_profile.py 8 128 1 > /dev/null 2>&1
python tools/ncu_source_top.py gpurun_out/cnn_fwd64.ncu-rep 30 > gpurun_out/cnn_fwd64_src.txt 2>&1
ncu -i gpurun_out/cnn_fwd64.ncu-rep --page details --csv > gpurun_out/cnn_fwd64_details.csv 2>&1
rm -f gpurun_out/*.ncu-rep
python tools/cnn_step_profile.py 8 128 5
DSX_CONV_2SM=0 python tools/cnn_step_profile.py 8 128 5
