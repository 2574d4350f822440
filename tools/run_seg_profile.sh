mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/sp_plain.log 2>&1 && DSX_NOISE_PIPELINE=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mt_segment_kernel" -s 4 -c 1 -o gpurun_out/seg_v4 $CMD > gpurun_out/sp_ncu.log 2>&1; echo sp=$?
