#!/bin/bash
# GPU suite + smoke (4 GPUs)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/f4_pytest_gpu.log 2>&1; tail -2 gpurun_out/f4_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f4_smoke.log 2>&1; tail -2 gpurun_out/f4_smoke.log
