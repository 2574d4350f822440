mkdir -p gpurun_out
N=${1:-2}
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29631 bench.py --gpus $N --steps 20 --warmup 3 > gpurun_out/e2emg_n$N.log 2>&1; echo bench_n$N=$?
tail -1 gpurun_out/e2emg_n$N.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'])"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k step_host > gpurun_out/e2emg_t.log 2>&1; echo t=$?; tail -1 gpurun_out/e2emg_t.log
