mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/bc_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/bc_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/bc_smoke.log 2>&1; echo smoke=$?
for nb in 1 4 8; do
DSX_NOISE_BATCH=$nb timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bc_b$nb.log 2>&1; echo b$nb=$?
tail -1 gpurun_out/bc_b$nb.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['step_breakdown_ms'])"
done
