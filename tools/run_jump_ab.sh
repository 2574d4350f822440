mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "engine or oracle or step_host" > gpurun_out/ja_parity.log 2>&1; echo parity=$?; tail -2 gpurun_out/ja_parity.log
for cfg in "1 4" "2 4" "2 8" "1 4" "2 4" "2 8"; do set -- $cfg
DSX_JUMP=$1 DSX_JUMP_PARTS=$2 timeout 300 python bench.py --steps 60 --warmup 8 --no-cpu-baseline --no-e2e > gpurun_out/ja_b.log 2>&1; echo jump$1_parts$2=$?
tail -1 gpurun_out/ja_b.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['noise_engine']['batched'])"
done
