# 4-GPU box: full GPU test suite (multi-rank parity at 2 and 4 GPUs) and the
# default bench line at N = 2 and 4 (as the driver's scaling run launches it)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/m4_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/m4_pytest.log
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n bench.py --gpus $n > gpurun_out/m4_bench_n$n.log 2>&1; echo bench_n$n=$?
  tail -1 gpurun_out/m4_bench_n$n.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['exposed_sync_frac'], d['sync_added_frac'], d['e2e']['value'], d['schedule']['synced_param_frac_per_step'])"
done
