#!/bin/bash
# ncu: update kernel with 2 local rows, noise-engine segment kernel, the
# cross-rank averaging kernel (2 GPUs in one process); overlap-group A/B at N=2
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
$NCU --set full --clock-control none --import-source on -k regex:lab_update_kernel -s 12 -c 1 -o gpurun_out/ncu_upd_k2 -f \
  python bench.py --workers 2 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_upd_k2.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:mt_segment_ws2 -s 4 -c 1 -o gpurun_out/ncu_seg -f \
  python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_seg.log 2>&1
$NCU --set full --clock-control none -k regex:p2p_average_kernel -c 2 -o gpurun_out/ncu_p2p2 -f \
  python -c "import ctypes as C,sys; sys.path.insert(0,'.'); from paper_2502_11058_b200 import native as N; e=C.c_double(); N.call('dsx_p2p_average_selftest', 2, 23379064, C.byref(e)); print(e.value)" > gpurun_out/ncu_p2p2.log 2>&1
for c in 2 3 6; do
  DSX_SYNC_CHUNKS=$c timeout 900 python bench.py --gpus 2 --no-e2e --no-cpu-baseline > gpurun_out/chunks_n2_c$c.json 2> gpurun_out/chunks_n2_c$c.err
done
# keep the transfer small: summaries + raw csv pages, reports removed
python tools/ncu_summary.py upd_k2:gpurun_out/ncu_upd_k2.ncu-rep seg_ws2:gpurun_out/ncu_seg.ncu-rep p2p_average_2gpu:gpurun_out/ncu_p2p2.ncu-rep > gpurun_out/r02_ncu_lab.md 2> gpurun_out/ncu_summary.err
for r in ncu_upd_k2 ncu_seg ncu_p2p2; do $NCU -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/$r.raw.csv 2>/dev/null; done
rm -f gpurun_out/*.ncu-rep
