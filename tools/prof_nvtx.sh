#!/bin/bash
# ncu --set full captures of chosen GEMM launches of ONE measured C4 step (NVTX range
# "measure" of bench.py --ncu).  PROF_IDS are indices among that step's coda_gemm_fast
# launches: 0 K4a, 1 K6, 2 K4b, 3 K7, 4 K9b, 5 wgrad qkv, 6 K10, 7 wgrad down, 8 K9a,
# 9 wgrad gate_up, 10 dgrad x, 11 wgrad out.  Output: gpurun_out/$PROF_DIR/prof_s<id>.ncu-rep
D=gpurun_out/${PROF_DIR:-r2}
mkdir -p $D
for s in ${PROF_IDS:-0 10}; do
  timeout -s KILL 400 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "measure/" \
    -k regex:coda_gemm_fast -s $s -c 1 -o $D/prof_s$s python bench.py --ncu --steps 1 --warmup 3 \
    ${BENCH_ARGS:-} > $D/prof_s$s.log 2>&1
  tail -2 $D/prof_s$s.log
done
ls -la $D
