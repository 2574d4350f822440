mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29631 tests/multigpu_parity.py > gpurun_out/mg4.log 2>&1; echo mg4=$?
grep -o '"results".*' gpurun_out/mg4.log
for w in 4 8; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2964$w bench.py --gpus 4 --steps 20 --warmup 3 --no-e2e --workers $w > gpurun_out/b12_n4_k$w.log 2>&1; echo n4k$w=$?
  tail -1 gpurun_out/b12_n4_k$w.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['exposed_sync_ms_per_iter'], d['sync_ms_per_iter'], d['roofline']['step_breakdown_ms'])"
done
