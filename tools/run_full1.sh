mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/f1_t.log 2>&1; echo pytest=$?; tail -2 gpurun_out/f1_t.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f1_smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/f1_smoke.log
timeout 300 python bench.py > gpurun_out/f1_b.log 2>&1; echo bench=$?
tail -1 gpurun_out/f1_b.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], d['ms_per_step'], r['frac'], r['kernel_ms'], d['e2e']['value'], d['clocks'])"
