#!/bin/bash
# A/B: update / engine SM partitions (green contexts) x single-coordinate bulk consumers, headline lab
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in "0 0" "0 1" "32 1" "40 1" "48 1" "56 1"; do
  set -- $cfg
  DSX_SM_SPLIT=$1 DSX_BULK_SINGLE=$2 timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ss$1_$2.json 2> gpurun_out/ss$1_$2.err
  python -c "import json; d=json.loads(open('gpurun_out/ss$1_$2.json').read().strip().splitlines()[-1]); r=d['roofline']; print('split=$1 single=$2', d['value'], d['ms_per_step'], r['kernel_ms'], r['achieved'], r['noise_engine']['batched']['per_step_ms'])" 2>&1 | tail -1
done
DSX_BULK_SINGLE=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_config1.py -q -x -p no:cacheprovider 2>&1 | tail -2
