#!/bin/bash
# NCCL env A/B on the 2-GPU MLP step (per-layer averages of 1-4 MB)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in "X=1" "NCCL_ALGO=NVLS" "NCCL_NVLS_ENABLE=0" "NCCL_ALGO=Ring NCCL_PROTO=LL128" "NCCL_ALGO=Ring NCCL_PROTO=LL" "NCCL_MIN_NCHANNELS=32" "NCCL_ALGO=Tree"; do
  env $cfg timeout 200 python bench.py --config mlp --gpus 2 --no-cpu-baseline --no-e2e > gpurun_out/ncclab.json 2> gpurun_out/ncclab.err
  python -c "import json;d=json.loads(open('gpurun_out/ncclab.json').read().strip().splitlines()[-1]);print('$cfg', d['value'], d['ms_per_step'], d.get('sync_added_ms_per_iter'), d['schedule']['profile_ms']['comm'][:3])" 2>&1 | tail -1
done
