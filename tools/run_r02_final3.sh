#!/bin/bash
# round-2 closing evidence (4 GPUs): GPU suite, smoke, NN bench lines after PDL, headline lab line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/f5_pytest_gpu.log 2>&1; tail -2 gpurun_out/f5_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f5_smoke.log 2>&1; tail -2 gpurun_out/f5_smoke.log
timeout 600 python bench.py > gpurun_out/f5_lab_n1.json 2> gpurun_out/f5_lab_n1.err
timeout 600 python bench.py --config mlp > gpurun_out/f5_mlp_n1.json 2> gpurun_out/f5_mlp_n1.err
for n in 2 4; do timeout 600 python bench.py --config mlp --gpus $n --no-cpu-baseline > gpurun_out/f5_mlp_n$n.json 2> gpurun_out/f5_mlp_n$n.err; done
for n in 1 4; do timeout 600 python bench.py --config resnet18_cnn --gpus $n --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/f5_cnn_n$n.json 2> gpurun_out/f5_cnn_n$n.err; done
timeout 600 python bench.py --config mlp_wide --no-cpu-baseline > gpurun_out/f5_mlpw_n1.json 2> gpurun_out/f5_mlpw_n1.err
timeout 900 python bench.py --config llama_mlp --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/f5_llama_n1.json 2> gpurun_out/f5_llama_n1.err
for f in gpurun_out/f5_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d.get('value'), d.get('ms_per_step'), (d.get('e2e') or {}).get('value'), d.get('exposed_sync_frac'), (d.get('roofline') or {}).get('achieved'))" 2>&1 | tail -1; done
