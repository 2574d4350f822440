#!/bin/bash
# multi-rank MLP: compute-only step graphs + eager NCCL averages (2 GPUs)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
DSX_TEST_GRAPHS=1 timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29733 tests/multigpu_mlp.py > gpurun_out/hy_test.log 2>&1; echo "graphs test rc=$?"; grep -o '"pass": [a-z]*' gpurun_out/hy_test.log
timeout 200 python bench.py --config mlp --gpus 2 --no-cpu-baseline > gpurun_out/hy_mlp_n2.json 2> gpurun_out/hy_mlp_n2.err; echo rc=$?
python -c "import json;d=json.loads(open('gpurun_out/hy_mlp_n2.json').read().strip().splitlines()[-1]);print('n2',d['value'],d['ms_per_step'],d.get('exposed_sync_frac'),d['e2e']['value'])"
timeout 300 python -m pytest tests/test_gpu_multigpu_nn.py -q -k mlp -p no:cacheprovider 2>&1 | tail -2
