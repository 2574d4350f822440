mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/sr_t4.log 2>&1; echo tests_r4=$?; tail -1 gpurun_out/sr_t4.log
DSX_SEG_R=6 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/sr_t6.log 2>&1; echo tests_r6=$?; tail -1 gpurun_out/sr_t6.log
for r in 4 6 4 6; do
DSX_SEG_R=$r timeout 300 python bench.py --steps 100 --warmup 8 --no-cpu-baseline --no-e2e > gpurun_out/sr.log 2>&1; echo r$r=$?
tail -1 gpurun_out/sr.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], d['ms_per_step'], r['noise_engine']['batched'])"
done
