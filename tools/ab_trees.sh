#!/bin/bash
# Alternate the whole-step bench between this tree and another source tree (same box).
# usage: bash tools/ab_trees.sh <other tree> [rounds] [extra bench args...]
B=$1; R=${2:-3}; shift 2
for r in $(seq $R); do
  for t in . $B; do
    echo "== $t round $r"
    (cd $t && timeout -s KILL 300 python bench.py --no-cpu --no-parity --ab-rounds 0 --steps 20 "$@" 2>/dev/null | tail -1)
  done
done
