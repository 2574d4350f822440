# Engine batch length A/B (N=1, sigma=1): it/s and engine ms/step per T.
# usage: bash tools/run_batch_ab.sh [T ...]   (default 4 6 8)
mkdir -p gpurun_out
BATCHES=${*:-4 6 8}
for rep in 1 2; do for nb in $BATCHES; do
DSX_NOISE_BATCH=$nb timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/ba.log 2>&1; echo nb$nb=$?
tail -1 gpurun_out/ba.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], d['ms_per_step'], r['noise_engine']['batched']['per_step_ms'])"
done; done
