mkdir -p gpurun_out
for nb in 4 8; do for pr in 1 0; do
DSX_NOISE_BATCH=$nb DSX_NOISE_PRIO=$pr timeout 300 python bench.py --steps 80 --warmup 8 --no-cpu-baseline --no-e2e > gpurun_out/ps_b${nb}_p$pr.log 2>&1; echo b${nb}p$pr=$?
tail -1 gpurun_out/ps_b${nb}_p$pr.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['noise_engine']['batched'])"
done; done
