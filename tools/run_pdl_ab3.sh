#!/bin/bash
# A/B: PDL across the conv-stack step chain; NN/conv GPU tests (2 GPUs)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 1 2; do for pdl in 0 1; do
  DSX_PDL=$pdl timeout 300 python bench.py --config resnet18_cnn --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pdl3.json 2> gpurun_out/pdl3.err
  python -c "import json; d=json.loads(open('gpurun_out/pdl3.json').read().strip().splitlines()[-1]); print('pdl=$pdl cnn n1', d['value'], d['ms_per_step'])" 2>&1 | tail -1
done; done
timeout 900 python -m pytest tests/test_gpu_nn.py tests/test_gpu_cnn.py tests/test_gpu_multigpu_nn.py tests/test_gpu_modes.py -q -x -p no:cacheprovider 2>&1 | tail -2
