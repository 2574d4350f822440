# Round evidence (one GPU): GPU tests + smoke, default bench line (as the
# driver runs it), reference arm, launch list, full ncu captures of the update
# kernel (sigma=0 and 1) and the noise engine kernels.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/ev_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/ev_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/ev_bench_default.log 2>&1; echo bench=$?
tail -1 gpurun_out/ev_bench_default.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/ev_bench_reference.log 2>&1; echo ref=$?
tail -1 gpurun_out/ev_bench_reference.log
timeout 300 python bench.py --sigma 0 --no-cpu-baseline > gpurun_out/ev_bench_sigma0.log 2>&1; echo bench0=$?
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/ev_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev_launches_sigma1.csv $CMD > /dev/null 2>&1; echo launches=$?
CMD0="python bench.py --steps 5 --warmup 3 --sigma 0 --no-cpu-baseline --no-e2e"
$CMD0 > gpurun_out/ev_plain0.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:lab_update -s 8 -c 2 -o gpurun_out/ev_update_sigma0 $CMD0 > /dev/null 2>&1; echo full0=$?
$CMD > gpurun_out/ev_plain1.log 2>&1 && DSX_NOISE_PIPELINE=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lab_update|mt_segment|mt_jump|mt_finish" -s 12 -c 4 -o gpurun_out/ev_engine_sigma1 $CMD > /dev/null 2>&1; echo full1=$?
