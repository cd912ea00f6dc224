#!/bin/bash
# Per-launch duration and SM clock of every fast GEMM in one C4 step (ncu), to compute
# efficiency against the MMA floor independently of the power-capped clock.
mkdir -p gpurun_out
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__cycles_elapsed.max \
   --clock-control none --nvtx --nvtx-include "measure/" --csv --log-file gpurun_out/ncu_eff.csv \
   python bench.py --ncu --steps 1 --warmup 1 > /dev/null 2>&1
python tools/eff_report.py gpurun_out/ncu_eff.csv
