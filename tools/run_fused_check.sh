mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multigpu.py -q -x > gpurun_out/fu_t0.log 2>&1; echo tests_default=$?; tail -1 gpurun_out/fu_t0.log
DSX_FUSED=1 timeout 900 python -m pytest tests/test_gpu_multigpu.py -q -x > gpurun_out/fu_t1.log 2>&1; echo tests_fused=$?; tail -1 gpurun_out/fu_t1.log
