#!/bin/bash
# NOTE: historical.  The "die" option (die-local rasters) was measured with this script and
# removed again because it did not reduce DRAM bytes (profiles/r01b_summary.md §5).
# Die-local rasters on vs off: DRAM bytes + duration of single launches (ncu), then
# interleaved timing of the same GEMMs and of the C4 step.
mkdir -p gpurun_out
for sh in ${SHAPES:-16384,4096,28672,0,1 4096,28672,16384,1,0 16384,28672,4096 14336,4096,16384,1,0}; do
  for d in 0 1; do
    echo "== $sh die=$d"
    CODA_DIE=$d timeout -s KILL 120 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_ltcfabric.sum \
      --clock-control none -k regex:coda_gemm_fast -s 2 -c 1 --csv python tools/gemm_bench.py --shape $sh --variant raster=8 --reps 1 2>/dev/null \
      | grep -E 'dram__bytes|gpu__time|ltcfabric'
  done
done
timeout -s KILL 300 python tools/gemm_bench.py --shape 16384,4096,28672,0,1 --shape 4096,28672,16384,1,0 --shape 16384,28672,4096 --variant die=0 --variant die=1 --reps 10
timeout -s KILL 300 python tools/ab_inproc.py --rounds 16 --variant die=0 --variant die=1
