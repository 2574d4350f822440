mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "oracle or engine" > gpurun_out/ac_t.log 2>&1; echo tests_default=$?
DSX_UPD_ASYNC=1 DSX_UPD_ASYNC_CTAS=74 timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "oracle or engine or step_host" > gpurun_out/ac_t2.log 2>&1; echo tests_async74=$?; tail -1 gpurun_out/ac_t2.log
for cfg in "0 0" "1 0" "1 148" "1 96" "1 74" "1 48"; do set -- $cfg
DSX_UPD_ASYNC=$1 DSX_UPD_ASYNC_CTAS=$2 timeout 300 python bench.py --steps 60 --warmup 8 --no-cpu-baseline --no-e2e > gpurun_out/ac.log 2>&1; echo async$1_ctas$2=$?
tail -1 gpurun_out/ac.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], d['ms_per_step'], r['frac'], r['step_breakdown_ms'])"
done
