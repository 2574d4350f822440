mkdir -p gpurun_out
for i in 1 2 3; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2978$i bench.py --gpus 4 --steps 100 --warmup 5 --no-e2e > gpurun_out/n4r.log 2>&1; echo run$i=$?
  tail -1 gpurun_out/n4r.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['ms_per_step_without_sync'], d['sync_added_frac'], d['schedule']['synced_param_frac_per_step'])"
done
