#!/bin/bash
# One measured C4 step under ncu: per-launch duration, SM clock, tensor-pipe utilisation and
# DRAM bytes; then the unfused cuBLAS+elementwise step's DRAM bytes for comparison.
# Report: python tools/ncu_tensor_report.py gpurun_out/ncu_tensor_c4.csv gpurun_out/launch_tags_c4.json
mkdir -p gpurun_out
M=gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum
timeout -s KILL 600 ncu --metrics $M --clock-control none --nvtx --nvtx-include "measure/" --csv \
   --log-file gpurun_out/ncu_tensor_c4.csv python bench.py --ncu --steps 1 --warmup 1 > /dev/null 2>&1
M2=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout -s KILL 600 ncu --metrics $M2 --clock-control none --nvtx --nvtx-include "measure/" --csv \
   --log-file gpurun_out/ncu_bytes_fused_c4.csv python tools/unfused_block.py --config c4 --ncu fused > /dev/null 2>&1
timeout -s KILL 600 ncu --metrics $M2 --clock-control none --nvtx --nvtx-include "measure/" --csv \
   --log-file gpurun_out/ncu_bytes_unfused_c4.csv python tools/unfused_block.py --config c4 --ncu unfused > /dev/null 2>&1
wc -l gpurun_out/ncu_tensor_c4.csv gpurun_out/ncu_bytes_*.csv
