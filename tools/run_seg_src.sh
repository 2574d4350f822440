# ncu --set full with source counters of the default segment kernel
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
DSX_NOISE_PIPELINE=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mt_segment_ws2_kernel" -s 2 -c 1 -o gpurun_out/seg_ws2 $CMD > gpurun_out/seg_ws2.log 2>&1; echo ncu=$?
