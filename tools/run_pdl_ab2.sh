#!/bin/bash
# A/B: PDL on every kernel of the MLP step chain (GEMMs + colsum/optimizer/softmax/loss/load_x), 2 GPUs
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 1 2; do for pdl in 0 1; do
  DSX_PDL=$pdl timeout 300 python bench.py --config mlp --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/pdl2.json 2> gpurun_out/pdl2.err
  python -c "import json; d=json.loads(open('gpurun_out/pdl2.json').read().strip().splitlines()[-1]); print('pdl=$pdl mlp n1', d['value'], d['ms_per_step'])" 2>&1 | tail -1
done; done
for pdl in 0 1; do
  DSX_PDL=$pdl timeout 300 python bench.py --config mlp --gpus 2 --no-cpu-baseline --no-e2e > gpurun_out/pdl2.json 2> gpurun_out/pdl2.err
  python -c "import json; d=json.loads(open('gpurun_out/pdl2.json').read().strip().splitlines()[-1]); print('pdl=$pdl mlp n2', d['value'], d['ms_per_step'])" 2>&1 | tail -1
done
timeout 900 python -m pytest tests/test_gpu_nn.py tests/test_gpu_cnn.py tests/test_gpu_multigpu_nn.py tests/test_gpu_modes.py -q -x -p no:cacheprovider 2>&1 | tail -2
