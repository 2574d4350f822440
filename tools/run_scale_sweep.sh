mkdir -p gpurun_out
N=${1:-4}
timeout 200 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/sw_n1.log 2>&1
tail -1 gpurun_out/sw_n1.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print('N=1', d['value'], d['ms_per_step'], d['roofline']['step_breakdown_ms'])"
for n in 2 $N; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2967$n bench.py --gpus $n --steps 20 --warmup 3 --no-e2e > gpurun_out/sw_n$n.log 2>&1
  tail -1 gpurun_out/sw_n$n.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print('N=$n', d['value'], d['ms_per_step'], d['exposed_sync_ms_per_iter'], d['sync_ms_per_iter'], d['roofline']['step_breakdown_ms'])"
done
