mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 tests/multigpu_parity.py > gpurun_out/mg2_log.log 2>&1; echo mg2=$?
tail -2 gpurun_out/mg2_log.log
timeout 300 python -m pytest tests/test_gpu_modes.py tests/test_gpu_parity.py -q -x > gpurun_out/modes2.log 2>&1; echo modes=$?; tail -3 gpurun_out/modes2.log
