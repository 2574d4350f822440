#!/bin/bash
# A/B: programmatic dependent launch of the tcgen05 GEMM / conv kernels (MLP, conv stack, wide MLP)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 1 2; do for pdl in 0 1; do
  for cfg in mlp resnet18_cnn mlp_wide; do
    DSX_PDL=$pdl timeout 300 python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pdl.json 2> gpurun_out/pdl.err
    python -c "import json; d=json.loads(open('gpurun_out/pdl.json').read().strip().splitlines()[-1]); print('pdl=$pdl $cfg', d['value'], d['ms_per_step'])" 2>&1 | tail -1
  done
done; done
timeout 900 python -m pytest tests/test_gpu_nn.py tests/test_gpu_cnn.py -q -x -p no:cacheprovider 2>&1 | tail -2
