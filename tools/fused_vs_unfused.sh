#!/bin/bash
# Whole C4 block, fused vs the unfused cuBLAS + torch elementwise sequence: timing line,
# and per-launch DRAM bytes of one step of each under ncu (north star "epilogue HBM
# bytes avoided versus an unfused cuBLAS-plus-elementwise sequence").
D=gpurun_out/${OUT_DIR:-fvu}
mkdir -p $D
for c in c4 c3; do
  timeout -s KILL 300 python tools/unfused_block.py --config $c > $D/unfused_vs_fused_$c.json 2>$D/unfused_$c.err
  for p in fused unfused; do
    timeout -s KILL 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none --nvtx --nvtx-include "measure/" --csv --log-file $D/ncu_bytes_${p}_$c.csv \
      python tools/unfused_block.py --config $c --ncu $p > /dev/null 2>&1
  done
done
ls $D
