#!/bin/bash
# DRAM bytes per tile vs the number of waves (M) for the K9a shape family: does re-read
# traffic accumulate with waves (drift between the consumers of a panel)?
for m in 2048 4096 8192 16384; do
  echo "== m=$m"
  timeout -s KILL 120 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none \
    -k regex:coda_gemm_fast -s 2 -c 1 --csv python tools/gemm_bench.py --shape $m,4096,28672,0,1 --variant raster=8 --reps 1 2>/dev/null \
    | grep -E 'dram__bytes|gpu__time'
done
