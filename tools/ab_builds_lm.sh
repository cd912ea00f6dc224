#!/bin/bash
# LM-head benchmark alternated between two source trees (build A/B on one box).
A=$1; B=$2; R=${3:-3}
for r in $(seq $R); do
  for t in $A $B; do
    echo "== $t"; timeout -s KILL 120 python $t/tools/lm_head_bench.py | cut -c1-160
  done
done
