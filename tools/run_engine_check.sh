mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "noise or oracle or smoke or steps" > gpurun_out/ec.log 2>&1; echo pytest=$?; tail -2 gpurun_out/ec.log
timeout 200 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ec_b.log 2>&1
tail -1 gpurun_out/ec_b.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['step_breakdown_ms'])"
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
DSX_NOISE_PIPELINE=0 timeout 600 ncu --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none -k regex:mt_ -c 12 --csv --log-file gpurun_out/ec.csv $CMD > /dev/null 2>&1; echo ncu=$?
