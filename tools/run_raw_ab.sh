mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q > gpurun_out/ra_parity.log 2>&1; echo parity=$?; tail -2 gpurun_out/ra_parity.log
DSX_NOISE_RAW=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "oracle or engine or smoke or steps" > gpurun_out/ra_parity1.log 2>&1; echo parity_raw=$?; tail -2 gpurun_out/ra_parity1.log
for cfg in 0 1 0 1; do
DSX_NOISE_RAW=$cfg timeout 300 python bench.py --steps 60 --warmup 8 --no-cpu-baseline --no-e2e > gpurun_out/ra_b.log 2>&1; echo raw$cfg=$?
tail -1 gpurun_out/ra_b.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], d['ms_per_step'], r['frac'], r['step_breakdown_ms'], r['noise_engine']['batched']['per_step_ms'])"
done
