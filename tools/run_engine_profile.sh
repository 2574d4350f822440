# ncu --set full (source counters) of the noise engine + sigma=1 update kernel
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/ep_plain.log 2>&1; echo plain=$?
tail -1 gpurun_out/ep_plain.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['roofline']['step_breakdown_ms'])"
DSX_NOISE_PIPELINE=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mt_segment_ws_kernel|mt_jump_kernel|lab_update_kernel|mt_finish" -s 8 -c 4 -o gpurun_out/engine_full $CMD > gpurun_out/ep_ncu.log 2>&1; echo ncu=$?
