#!/bin/bash
# Full ncu captures (one launch each) of the epilogue-heavy K10, K6, K7 and the lean K4b in the C4 step.
# fast-kernel launch order in a step: 0 K4a, 1 K6, 2 K4b, 3 K7, 4 K9b, 5 wgrad_qkv, 6 K10, 7 wgrad_down, 8 K9a, ...
mkdir -p gpurun_out
for spec in "k6:1" "k4b:2" "k7:3" "k10:6"; do
  name=${spec%%:*}; skip=${spec##*:}
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:coda_gemm_fast -s $skip -c 1 \
      -o gpurun_out/prof2_$name python bench.py --ncu --steps 0 --warmup 1 > gpurun_out/ncu2_$name.log 2>&1
  tail -1 gpurun_out/ncu2_$name.log
done
