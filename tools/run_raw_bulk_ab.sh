#!/bin/bash
# A/B: engine normals + bulk update vs raw attempts + bulk update doing the polar transform
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 1 2; do for raw in 0 1; do
  DSX_NOISE_RAW=$raw timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/raw$raw.$r.json 2> gpurun_out/raw$raw.$r.err
  python -c "import json; d=json.loads(open('gpurun_out/raw$raw.$r.json').read().strip().splitlines()[-1]); r=d['roofline']; print('raw=$raw', d['value'], d['ms_per_step'], r['kernel_ms'], r['achieved'], r['noise_engine']['batched']['per_step_ms'])" 2>&1 | tail -1
done; done
DSX_NOISE_RAW=1 timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/raw1_parity.json 2> gpurun_out/raw1_parity.err
python -c "import json; d=json.loads(open('gpurun_out/raw1_parity.json').read().strip().splitlines()[-1]); print('parity', d.get('parity'))"
DSX_NOISE_RAW=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_config1.py -q -x -p no:cacheprovider 2>&1 | tail -2
