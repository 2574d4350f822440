mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29582 tools/sync_probe.py > gpurun_out/sp4.log 2>&1; echo sp4=$?; tail -1 gpurun_out/sp4.log
for s in 1 0; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2967$s bench.py --gpus 4 --steps 30 --warmup 5 --no-e2e --sigma $s > gpurun_out/ms_n4_s$s.log 2>&1; echo n4s$s=$?
  tail -1 gpurun_out/ms_n4_s$s.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); sc=d['schedule']; t=sc.pop('text',None); print(d['value'], d['ms_per_step'], d['exposed_sync_ms_per_iter'], d['sync_ms_per_iter'], d['exposed_sync_frac'], json.dumps(sc), d['roofline']['step_breakdown_ms'])"
done
