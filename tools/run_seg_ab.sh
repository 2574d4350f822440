# A/B of segment-kernel variants: parity tests on the default, bench on each
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/ab_parity.log 2>&1; echo parity=$?; tail -2 gpurun_out/ab_parity.log
for v in 1 2; do
  DSX_SEG_WS=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_ws$v.log 2>&1; echo ws$v=$?
  tail -1 gpurun_out/ab_ws$v.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['roofline']['step_breakdown_ms'])"
done
DSX_NOISE_PIPELINE=0 timeout 600 ncu --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none -k regex:mt_ -c 8 --csv --log-file gpurun_out/ab_launch.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu=$?
