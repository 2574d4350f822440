mkdir -p gpurun_out
for nb in 2 3 4 6; do
DSX_NOISE_BATCH=$nb timeout 300 python bench.py --steps 60 --warmup 8 --no-cpu-baseline --no-e2e > gpurun_out/bs_b$nb.log 2>&1; echo b$nb=$?
tail -1 gpurun_out/bs_b$nb.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['noise_engine']['batched'])"
done
