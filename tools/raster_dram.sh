#!/bin/bash
# DRAM bytes and duration of one plain GEMM launch per raster group (ncu, single launch each).
mkdir -p gpurun_out
SHAPES=${SHAPES:-"16384,4096,28672,0,1 4096,28672,16384,1,0 16384,28672,4096"}
for sh in $SHAPES; do
  for g in ${GROUPS_:-2 4 8 16 32}; do
    CODA_RASTER_GROUP=$g timeout -s KILL 120 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_op_read_hit_rate.pct \
      --clock-control none -k regex:coda_gemm_fast -s 2 -c 1 --csv python tools/gemm_bench.py --shape $sh --variant raster=$g --reps 1 2>/dev/null \
      | grep -E 'dram__bytes|gpu__time|hit_rate' | awk -F'","' -v sh=$sh -v g=$g '{gsub(/"/,"",$NF); printf "%s g=%s %s %s %s\n", sh, g, $(NF-2), $(NF-1), $NF}'
  done
done
