mkdir -p gpurun_out
DSX_UPD_BULK=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "oracle or engine or smoke or step_host or external" > gpurun_out/bk_t.log 2>&1; echo tests_bulk=$?; tail -3 gpurun_out/bk_t.log
for cfg in 0 1 96 74; do
DSX_UPD_BULK=$cfg timeout 200 python bench.py --steps 60 --warmup 8 --no-cpu-baseline --no-e2e > gpurun_out/bk.log 2>&1; echo bulk$cfg=$?
tail -1 gpurun_out/bk.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], d['ms_per_step'], r['frac'], r['step_breakdown_ms'])"
done
DSX_UPD_BULK=1 timeout 200 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --sigma 0 > gpurun_out/bk0.log 2>&1; echo bulk_s0=$?
tail -1 gpurun_out/bk0.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], d['ms_per_step'], r['frac'])"
