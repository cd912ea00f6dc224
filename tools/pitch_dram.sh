#!/bin/bash
# DRAM bytes / duration of one plain GEMM launch vs the operands' row-pitch padding (ncu).
mkdir -p gpurun_out
for sh in ${SHAPES:-16384,4096,28672,0,1 4096,28672,16384,1,0 16384,28672,4096}; do
  for pad in ${PADS:-0 8 64 128}; do
    echo "== $sh pad=$pad"
    timeout -s KILL 120 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_op_read_hit_rate.pct \
      --clock-control none -k regex:coda_gemm_fast -s 2 -c 1 --csv python tools/gemm_bench.py --shape $sh --variant raster=8 --reps 1 --pad $pad 2>/dev/null \
      | grep -E 'dram__bytes|gpu__time|hit_rate'
  done
done
