#!/bin/bash
# round-2 end evidence, third pass (4 GPUs): GPU suite, smoke, bench lines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/f3_pytest_gpu.log 2>&1; tail -2 gpurun_out/f3_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f3_smoke.log 2>&1; tail -2 gpurun_out/f3_smoke.log
for n in 1 2 4; do timeout 600 python bench.py --gpus $n > gpurun_out/f3_lab_n$n.json 2> gpurun_out/f3_lab_n$n.err; done
timeout 600 python bench.py --impl reference > gpurun_out/f3_lab_ref.json 2> gpurun_out/f3_lab_ref.err
timeout 600 python bench.py --config mlp > gpurun_out/f3_mlp_n1.json 2> gpurun_out/f3_mlp_n1.err
for n in 2 4; do timeout 600 python bench.py --config mlp --gpus $n --no-cpu-baseline > gpurun_out/f3_mlp_n$n.json 2> gpurun_out/f3_mlp_n$n.err; done
for n in 1 2 4; do timeout 600 python bench.py --config resnet18_cnn --gpus $n --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/f3_cnn_n$n.json 2> gpurun_out/f3_cnn_n$n.err; done
timeout 600 python bench.py --config mlp_wide --gpus 4 --no-cpu-baseline > gpurun_out/f3_mlpw_n4.json 2> gpurun_out/f3_mlpw_n4.err
for f in gpurun_out/f3_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d.get('value'), d.get('ms_per_step'), (d.get('e2e') or {}).get('value'), d.get('exposed_sync_frac'))" 2>&1 | tail -1; done
