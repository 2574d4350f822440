mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q > gpurun_out/as_parity.log 2>&1; echo parity=$?; tail -2 gpurun_out/as_parity.log
for cfg in "1 1" "0 1" "1 0" "0 0"; do set -- $cfg
DSX_UPD_ASYNC=$1 DSX_NOISE_RAW=$2 timeout 300 python bench.py --steps 60 --warmup 8 --no-cpu-baseline --no-e2e > gpurun_out/as_b.log 2>&1; echo async$1_raw$2=$?
tail -1 gpurun_out/as_b.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], d['ms_per_step'], r['frac'], r['step_breakdown_ms'], r['noise_engine']['batched']['per_step_ms'])"
done
DSX_UPD_ASYNC=1 timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --sigma 0 > gpurun_out/as_b0.log 2>&1; echo s0=$?
tail -1 gpurun_out/as_b0.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], d['ms_per_step'], r['frac'], r['step_breakdown_ms'])"
