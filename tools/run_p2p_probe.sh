mkdir -p gpurun_out
N=${1:-2}
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2958$N tools/sync_probe.py > gpurun_out/pp_n$N.log 2>&1; echo sp=$?; tail -1 gpurun_out/pp_n$N.log | python3 -c "
import sys,json; d=json.loads(sys.stdin.read())
for k,v in d.items():
    if isinstance(v,dict) and 'serial' in v: print(k, v['serial']['sync_ms'], v['overlap']['sync_ms'])
print('nccl', d['torch_nccl_allreduce'])"
