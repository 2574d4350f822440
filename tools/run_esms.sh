mkdir -p gpurun_out
for e in 148 124 100 88 74 148 100 88; do
  DSX_ENGINE_SMS=$e timeout 300 python bench.py --steps 100 --warmup 8 --no-e2e --no-cpu-baseline > gpurun_out/es1.log 2>&1; echo N1_esms$e=$?
  tail -1 gpurun_out/es1.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['noise_engine']['batched']['per_step_ms'])"
done
for e in 88 74; do
  DSX_ENGINE_SMS=$e timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29794 bench.py --gpus 4 --steps 100 --warmup 5 --no-e2e > gpurun_out/es.log 2>&1; echo N4_esms$e=$?
  tail -1 gpurun_out/es.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['ms_per_step_without_sync'], d['sync_added_frac'], d['roofline']['noise_engine']['batched']['per_step_ms'])"
done
