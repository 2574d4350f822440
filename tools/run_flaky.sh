#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2 3 4 5 6; do timeout 120 python -m pytest tests/test_gpu_nn.py -q -k f32_gemm -p no:cacheprovider 2>&1 | tail -1; done
timeout 600 python -m pytest tests/test_gpu_nn.py -q -p no:cacheprovider 2>&1 | tail -2
timeout 300 python tools/pcie_multi_probe.py > gpurun_out/pcie_multi.json 2>&1; cat gpurun_out/pcie_multi.json
