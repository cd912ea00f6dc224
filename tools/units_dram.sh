#!/bin/bash
# NOTE: historical -- uses the measurement-only "units" option, removed afterwards (profiles/r01b_summary.md §5).
# DRAM bytes / duration of one plain GEMM launch vs the number of concurrently running
# CTA pairs (measurement-only option "units"): is the large-K re-read traffic a function
# of how many tiles run at once (drift between consumers of one panel), or of L2 capacity?
for sh in ${SHAPES:-16384,4096,28672,0,1 4096,28672,16384,1,0 16384,28672,4096}; do
  for u in 74 37 18 9; do
    echo "== $sh units=$u"
    CODA_UNITS=$u timeout -s KILL 120 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_op_read_hit_rate.pct \
      --clock-control none -k regex:coda_gemm_fast -s 2 -c 1 --csv python tools/gemm_bench.py --shape $sh --variant raster=8 --reps 1 2>/dev/null \
      | grep -E 'dram__bytes|gpu__time|hit_rate'
  done
done
