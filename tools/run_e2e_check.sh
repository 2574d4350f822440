mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/e2e_parity.log 2>&1; echo parity=$?; tail -3 gpurun_out/e2e_parity.log
for ch in 8 24 48; do
DSX_HOST_CHUNKS=$ch timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 10 > gpurun_out/e2e_b$ch.log 2>&1; echo b$ch=$?
tail -1 gpurun_out/e2e_b$ch.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'])"
done
