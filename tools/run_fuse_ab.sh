#!/bin/bash
# A/B: the 1-GPU MLP with each scheduled layer's average fused into its optimizer pass
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 1 2; do for f in 0 1; do
  DSX_FUSE_AVG=$f timeout 300 python bench.py --config mlp --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/fuse.json 2> gpurun_out/fuse.err
  python -c "import json; d=json.loads(open('gpurun_out/fuse.json').read().strip().splitlines()[-1]); print('fuse=$f mlp', d['value'], d['ms_per_step'])" 2>&1 | tail -1
  DSX_FUSE_AVG=$f timeout 300 python bench.py --config mlp_wide --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fuse.json 2> gpurun_out/fuse.err
  python -c "import json; d=json.loads(open('gpurun_out/fuse.json').read().strip().splitlines()[-1]); print('fuse=$f mlp_wide', d['value'], d['ms_per_step'], d['clocks']['reasons'])" 2>&1 | tail -1
done; done
timeout 900 python -m pytest tests/test_gpu_nn.py tests/test_gpu_modes.py -q -x -p no:cacheprovider 2>&1 | tail -2
