#!/bin/bash
# A/B: host-state step pipeline depth (DSX_HOST_CHUNKS) on the headline e2e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 1 2; do for c in 12 24 48 96; do
  DSX_HOST_CHUNKS=$c timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/hc.json 2> gpurun_out/hc.err
  python -c "import json; d=json.loads(open('gpurun_out/hc.json').read().strip().splitlines()[-1]); print('chunks=$c', d['value'], d['e2e']['value'])" 2>&1 | tail -1
done; done
