mkdir -p gpurun_out
N=${1:-2}
timeout 900 python -m pytest tests/test_gpu_multigpu.py -q -x > gpurun_out/fu_t.log 2>&1; echo tests=$?; tail -3 gpurun_out/fu_t.log
for s in 1 0; do for f in 1 0; do
  DSX_FUSED=$f timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 297$f$s bench.py --gpus $N --steps 60 --warmup 5 --no-e2e --sigma $s > gpurun_out/fu.log 2>&1; echo N${N}_s${s}_fused$f=$?
  tail -1 gpurun_out/fu.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['ms_per_step_without_sync'], d['sync_added_frac'], d['schedule']['synced_param_frac_per_step'], d['roofline']['kernel_ms'])"
done; done
