mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "step_host or cpp_api or acceptance" > gpurun_out/e2e_t.log 2>&1; echo tests=$?; tail -2 gpurun_out/e2e_t.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 20 > gpurun_out/e2e_b.log 2>&1; echo bench=$?
tail -1 gpurun_out/e2e_b.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'])"
