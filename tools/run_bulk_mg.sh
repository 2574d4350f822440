mkdir -p gpurun_out
N=${1:-2}
timeout 900 python -m pytest tests/test_gpu_multigpu.py -q -x > gpurun_out/bm_t.log 2>&1; echo tests=$?; tail -1 gpurun_out/bm_t.log
for n in 2 $N; do for b in -1 0; do
  DSX_UPD_BULK=$b timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2976$n bench.py --gpus $n --steps 60 --warmup 5 --no-e2e > gpurun_out/bm.log 2>&1; echo N${n}_bulk$b=$?
  tail -1 gpurun_out/bm.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], d['ms_per_step'], r['frac'], r['kernel_ms'], d['sync_added_frac'])"
done; done
