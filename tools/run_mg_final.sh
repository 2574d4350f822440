# multi-GPU: tests, default bench lines, throttled sweep
mkdir -p gpurun_out
N=${1:-4}
timeout 900 python -m pytest tests/test_gpu_multigpu.py -q > gpurun_out/mf_t.log 2>&1; echo tests=$?; tail -1 gpurun_out/mf_t.log
for n in 2 $N; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2964$n bench.py --gpus $n > gpurun_out/mf_bench_n$n.log 2>&1; echo bench_n$n=$?
  tail -1 gpurun_out/mf_bench_n$n.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['exposed_sync_frac'], d['sync_added_frac'], d['e2e']['value'], d['schedule']['synced_param_frac_per_step'])"
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2965$n tools/sweep.py --link-ratio 2 --out gpurun_out/sweep_throttled_n$n.json > gpurun_out/mf_sw_n$n.log 2>&1; echo sweep_t_n$n=$?
  grep '^{' gpurun_out/mf_sw_n$n.log | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['H'], d['L'], d['synced_param_frac_per_step'], d['plsgd']['it_per_s'], d['plsgd_no_fill']['it_per_s'], d['flsgd']['it_per_s'], d['speedup_vs_flsgd'], d['speedup_no_fill_vs_flsgd'], d['plsgd']['exposed_sync_frac'], d['flsgd']['exposed_sync_frac'])"
done
