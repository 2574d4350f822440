mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q > gpurun_out/sc_t.log 2>&1; echo tests=$?; tail -1 gpurun_out/sc_t.log
for i in 1 2; do
timeout 300 python bench.py --steps 100 --warmup 8 --no-cpu-baseline --no-e2e > gpurun_out/sc.log 2>&1; echo bench=$?
tail -1 gpurun_out/sc.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], d['ms_per_step'], r['step_breakdown_ms'], r['noise_engine']['batched'])"
done
DSX_NOISE_PIPELINE=0 timeout 600 ncu --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none -k regex:mt_segment -c 2 --csv --log-file gpurun_out/sc_ncu.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu=$?
