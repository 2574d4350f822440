mkdir -p gpurun_out
for pad in 0 90000 0 90000; do
DSX_SEG_PAD=$pad timeout 300 python bench.py --steps 60 --warmup 8 --no-cpu-baseline --no-e2e > gpurun_out/pad.log 2>&1; echo pad$pad=$?
tail -1 gpurun_out/pad.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], d['ms_per_step'], r['step_breakdown_ms'], r['noise_engine']['batched']['per_step_ms'])"
done
