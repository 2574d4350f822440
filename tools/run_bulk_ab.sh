#!/bin/bash
# A/B: bulk-copy update kernel for 1-4 local rows (chunk scaled by row count)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export DSX_FLAG_TIMEOUT_S=120
timeout 900 python -m pytest tests/test_gpu_multigpu.py -q --timeout 600 -k "p2p_average_kernel or bit_exact" > gpurun_out/bulk_tests.log 2>&1; echo "rc=$?" >> gpurun_out/bulk_tests.log
DSX_UPD_BULK=1 timeout 900 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_parity.py -q --timeout 600 -x > gpurun_out/bulk_tests_forced.log 2>&1; echo "rc=$?" >> gpurun_out/bulk_tests_forced.log
unset DSX_FLAG_TIMEOUT_S
for n in 2 4; do
  for b in 0 1; do
    DSX_UPD_BULK=$b timeout 900 python bench.py --gpus $n --no-e2e --no-cpu-baseline > gpurun_out/ab_n${n}_bulk$b.json 2> gpurun_out/ab_n${n}_bulk$b.err
  done
done
for b in 0 1; do
  DSX_UPD_BULK=$b timeout 900 python bench.py --workers 2 --no-e2e --no-cpu-baseline > gpurun_out/ab_k2_bulk$b.json 2> gpurun_out/ab_k2_bulk$b.err
done
