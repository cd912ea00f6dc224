#!/bin/bash
# Interleaved A/B of an environment toggle on the C4 bench: tools/ab_env.sh VAR valA valB [extra bench args]
VAR=$1; A=$2; B=$3; shift 3
for rep in 1 2; do
  for val in $A $B; do
    env $VAR=$val timeout -s KILL 600 python bench.py --steps 20 --warmup 3 --no-cpu "$@" > gpurun_out/ab_${VAR}_${val}_$rep.json 2>&1
    python - "$VAR" "$val" "$rep" <<'PY'
import json, sys
var, val, rep = sys.argv[1:4]
d = json.loads(open(f"gpurun_out/ab_{var}_{val}_{rep}.json").read().strip().splitlines()[-1])
print(f"{var}={val} rep{rep}: {d['value']:.0f} tok/s  {d['ms_per_step']:.3f} ms/step  clk {d['clocks']['sm_mhz']} "
      f"per-MHz {d['value']/max(1,d['clocks']['sm_mhz'] or 1):.1f}  e2e {d['e2e']['value']:.0f}")
PY
  done
done
