#!/bin/bash
# Alternate the same single-GEMM benchmark between two source trees (build A/B on one box).
# usage: bash tools/ab_builds.sh <treeA> <treeB> [rounds]
A=$1; B=$2; R=${3:-3}
for r in $(seq $R); do
  for t in $A $B; do
    echo "== $t round $r"
    timeout -s KILL 200 python $t/tools/gemm_bench.py --shape 16384,28672,4096 --shape 16384,4096,28672,0,1 --shape 4096,28672,16384,1,0 --variant raster=8 --reps 8 2>&1 | grep '^{'
  done
done
