mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/uc_parity.log 2>&1; echo parity=$?; tail -2 gpurun_out/uc_parity.log
for s in 1 0; do
timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --sigma $s > gpurun_out/uc_b$s.log 2>&1; echo b$s=$?
tail -1 gpurun_out/uc_b$s.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], d['ms_per_step'], r['achieved'], r['frac'], r['step_breakdown_ms'])"
done
DSX_NOISE_PIPELINE=0 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread --clock-control none -k regex:lab_update -c 4 --csv --log-file gpurun_out/uc_ncu.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu=$?
