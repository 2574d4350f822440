mkdir -p gpurun_out
N=${1:-2}
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29591 tools/sweep.py --out gpurun_out/sweep_n$N.json > gpurun_out/sweep_n$N.log 2>&1; echo sweep=$?
grep '^{' gpurun_out/sweep_n$N.log | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['H'], d['L'], d['synced_param_frac_per_step'], d['plsgd']['it_per_s'], d['plsgd_no_fill']['it_per_s'], d['flsgd']['it_per_s'], d['speedup_vs_flsgd'], d['speedup_no_fill_vs_flsgd'], d['plsgd']['exposed_sync_frac'], d['plsgd_no_fill']['exposed_sync_frac'], d['flsgd']['exposed_sync_frac'])"
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29593 tools/sweep.py --link-ratio 2 --out gpurun_out/sweep_throttled_n$N.json > gpurun_out/sweept_n$N.log 2>&1; echo sweep_throttled=$?
grep '^{' gpurun_out/sweept_n$N.log | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['H'], d['L'], d['synced_param_frac_per_step'], d['plsgd']['it_per_s'], d['plsgd_no_fill']['it_per_s'], d['flsgd']['it_per_s'], d['speedup_vs_flsgd'], d['speedup_no_fill_vs_flsgd'], d['plsgd']['exposed_sync_frac'], d['flsgd']['exposed_sync_frac'])"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29592 bench.py --gpus $N --steps 30 --warmup 5 --no-e2e > gpurun_out/bn_n$N.log 2>&1; echo bench=$?
tail -1 gpurun_out/bn_n$N.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['exposed_sync_frac'], d['averaging'])"
