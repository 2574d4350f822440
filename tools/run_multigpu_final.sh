# Multi-GPU round evidence: GPU tests on N GPUs (multi-rank parity included),
# then the default bench line at N GPUs as the driver launches it.
N=${1:-2}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rs > gpurun_out/final_pt_n$N.log 2>&1; echo pytest=$?; tail -3 gpurun_out/final_pt_n$N.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29661 bench.py --gpus $N > gpurun_out/final_bench_n$N.log 2>&1; echo bench=$?
tail -1 gpurun_out/final_bench_n$N.log
