mkdir -p gpurun_out
N=${1:-2}
timeout 600 python -m pytest tests/test_gpu_multigpu.py -x -q > gpurun_out/fb_mg.log 2>&1; echo mgtest=$?; tail -2 gpurun_out/fb_mg.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29583 tools/sync_probe.py > gpurun_out/fb_sp.log 2>&1; echo sp=$?; tail -1 gpurun_out/fb_sp.log
for s in 1 0; do
  for fbv in 1 0; do
  DSX_FLAG_BARRIER=$fbv timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2968$s bench.py --gpus $N --steps 30 --warmup 5 --no-e2e --sigma $s > gpurun_out/fb_n${N}_s${s}_f$fbv.log 2>&1; echo n${N}s${s}f$fbv=$?
  tail -1 gpurun_out/fb_n${N}_s${s}_f$fbv.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); sc=d['schedule']; t=sc.pop('text',None); print(d['value'], d['ms_per_step'], d['exposed_sync_ms_per_iter'], d['sync_ms_per_iter'], d['exposed_sync_frac'], json.dumps(sc))"
  done
done
