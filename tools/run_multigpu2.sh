mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pt2.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pt2.log
grep -o '"results".*' gpurun_out/pt2.log | head -2
for s in 0 1; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2965$s bench.py --gpus 2 --steps 20 --warmup 3 --no-e2e --sigma $s > gpurun_out/b13_n2_s$s.log 2>&1; echo n2s$s=$?
  tail -1 gpurun_out/b13_n2_s$s.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['exposed_sync_ms_per_iter'], d['sync_ms_per_iter'], d['roofline']['step_breakdown_ms'])"
done
