#!/bin/bash
# A/B the CTA-pair mainloop against the single-CTA one on the C4 bench (GPU box).
for cg in 1 2; do
  CODA_CG=$cg timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_cg$cg.json 2>&1
  python - "$cg" <<'PY'
import json, sys
cg = sys.argv[1]
line = open(f"gpurun_out/bench_cg{cg}.json").read().strip().splitlines()[-1]
d = json.loads(line)
print("CG", cg, "tok/s", round(d["value"]), "block TF/s", round(d["block_tflops"]), "clk", d["clocks"])
for k, v in d["launch_breakdown_ms"].items():
    print("   ", k, v)
PY
done
