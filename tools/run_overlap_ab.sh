# overlap group count A/B at N GPUs (sigma = 1), repeated
mkdir -p gpurun_out
N=${1:-2}; shift
for rep in 1 2; do for ch in "$@"; do
  DSX_SYNC_CHUNKS=$ch timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 298$ch$N bench.py --gpus $N --steps 100 --warmup 5 --no-e2e > gpurun_out/ov.log 2>&1; echo N${N}_chunks$ch=$?
  tail -1 gpurun_out/ov.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['ms_per_step_without_sync'], d['sync_ms_per_iter'], d['sync_added_frac'], d['schedule']['synced_param_frac_per_step'])"
done; done
