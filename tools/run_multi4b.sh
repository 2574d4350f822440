#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export DSX_FLAG_TIMEOUT_S=120
DSX_MLP_GRAPHS_NCCL=1 DSX_TEST_GRAPHS=1 timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29711 tests/multigpu_mlp.py > gpurun_out/nccl_graph2.log 2>&1; echo "rc=$?" >> gpurun_out/nccl_graph2.log
unset DSX_FLAG_TIMEOUT_S
for n in 2 4; do
  timeout 600 python bench.py --config mlp --gpus $n > gpurun_out/mlp4b_n$n.json 2> gpurun_out/mlp4b_n$n.err
done
if grep -q '"pass": true' gpurun_out/nccl_graph2.log; then
  for n in 2 4; do
    DSX_MLP_GRAPHS_NCCL=1 timeout 600 python bench.py --config mlp --gpus $n --no-cpu-baseline > gpurun_out/mlp4g_n$n.json 2> gpurun_out/mlp4g_n$n.err
  done
fi
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29721 tools/sweep.py --out gpurun_out/sweep_n4.json > gpurun_out/sweep_n4.log 2>&1
