#!/bin/bash
# NOTE: historical -- the l2hint option was removed after this measurement (profiles/r01b_summary.md §5).
# Operand L2 eviction hints (option l2hint): DRAM bytes + duration per single launch (ncu),
# then interleaved timing of the GEMMs and of the C4 step.
for sh in ${SHAPES:-16384,4096,28672,0,1 4096,28672,16384,1,0 16384,28672,4096}; do
  for h in 0 1 2 3; do
    echo "== $sh l2hint=$h"
    CODA_L2HINT=$h timeout -s KILL 120 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum \
      --clock-control none -k regex:coda_gemm_fast -s 2 -c 1 --csv python tools/gemm_bench.py --shape $sh --variant raster=8 --reps 1 2>/dev/null \
      | grep -E 'dram__bytes|gpu__time'
  done
done
timeout -s KILL 300 python tools/gemm_bench.py --shape 16384,4096,28672,0,1 --shape 4096,28672,16384,1,0 --shape 16384,28672,4096 --variant l2hint=0 --variant l2hint=1 --variant l2hint=2 --variant l2hint=3 --reps 8
timeout -s KILL 300 python tools/ab_inproc.py --rounds 12 --variant l2hint=0 --variant l2hint=1 --variant l2hint=2 --variant l2hint=3
