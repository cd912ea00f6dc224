#!/bin/bash
# NOTE: historical -- the wave_sync option was removed after this measurement (profiles/r01b_summary.md §5).
# Wave sync on vs off: DRAM bytes + duration of single large-K launches (ncu), then the
# interleaved C4 step.
for sh in ${SHAPES:-16384,4096,28672,0,1 4096,28672,16384,1,0 16384,4096,14336 14336,4096,16384,1,0}; do
  for v in ${VALS:-0 50 75 95}; do
    echo "== $sh wave_sync=$v"
    CODA_WAVE_SYNC=$v timeout -s KILL 120 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum \
      --clock-control none -k regex:coda_gemm_fast -s 2 -c 1 --csv python tools/gemm_bench.py --shape $sh --variant raster=8 --reps 1 2>/dev/null \
      | grep -E 'dram__bytes|gpu__time'
  done
done
timeout -s KILL 300 python tools/gemm_bench.py --shape 16384,4096,28672,0,1 --shape 4096,28672,16384,1,0 --variant wave_sync=0 --variant wave_sync=50 --variant wave_sync=75 --variant wave_sync=95 --reps 10
timeout -s KILL 400 python tools/ab_inproc.py --rounds 20 --variant wave_sync=0 --variant wave_sync=50 --variant wave_sync=75 --variant wave_sync=95
