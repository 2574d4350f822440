# overlap granularity A/B at N GPUs: it/s, classic exposed fraction, and the
# sync time an iteration actually pays (vs the same steps with nothing synced)
mkdir -p gpurun_out
N=${1:-2}
for s in 1 0; do
for ch in 1 4; do
  DSX_SYNC_CHUNKS=$ch timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 297$s$ch bench.py --gpus $N --steps 40 --warmup 5 --no-e2e --sigma $s > gpurun_out/ov.log 2>&1; echo N${N}_s${s}_chunks$ch=$?
  tail -1 gpurun_out/ov.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['ms_per_step_without_sync'], d['sync_ms_per_iter'], d['exposed_sync_frac'], d['sync_added_frac'], d['schedule']['synced_param_frac_per_step'])"
done; done
