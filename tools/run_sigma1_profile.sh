timeout 300 python bench.py --steps 30 --warmup 3 --sigma 1 --no-cpu-baseline > gpurun_out/b11_s1.log 2>&1
tail -1 gpurun_out/b11_s1.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['achieved'], d['roofline']['frac'], d['roofline']['step_breakdown_ms'], d['e2e'])"
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
DSX_NOISE_PIPELINE=0 timeout 600 ncu --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none -k regex:mt_ -c 12 --csv --log-file gpurun_out/l11.csv $CMD > /dev/null 2>&1; echo l11=$?
