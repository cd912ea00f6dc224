#!/bin/bash
# One GPU-box session: parity tests, C2 primitive sweep, fused-vs-unfused block, C3/C5 benches,
# and ncu dram-byte captures of one fused step and one unfused step (C4).
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -6
timeout -s KILL 300 python tools/primitive_sweep.py > gpurun_out/c2_sweep.jsonl 2>&1; cat gpurun_out/c2_sweep.jsonl | cut -c1-300
timeout -s KILL 300 python tools/unfused_block.py --config c4 > gpurun_out/unfused_c4.json 2>&1; cat gpurun_out/unfused_c4.json | cut -c1-600
timeout -s KILL 300 python tools/unfused_block.py --config c3 > gpurun_out/unfused_c3.json 2>&1; cat gpurun_out/unfused_c3.json | cut -c1-600
timeout -s KILL 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_c3.json 2>&1; tail -c 700 gpurun_out/bench_c3.json
timeout -s KILL 600 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c5.json 2>&1; tail -c 700 gpurun_out/bench_c5.json
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout -s KILL 600 ncu --metrics $M --clock-control none --nvtx --nvtx-include "measure/" --csv --log-file gpurun_out/ncu_bytes_fused_c4.csv python tools/unfused_block.py --config c4 --ncu fused > /dev/null 2>&1
timeout -s KILL 600 ncu --metrics $M --clock-control none --nvtx --nvtx-include "measure/" --csv --log-file gpurun_out/ncu_bytes_unfused_c4.csv python tools/unfused_block.py --config c4 --ncu unfused > /dev/null 2>&1
timeout -s KILL 600 ncu --metrics $M --clock-control none --nvtx --nvtx-include "measure/" --csv --log-file gpurun_out/ncu_bytes_c2.csv python tools/primitive_sweep.py --ncu > /dev/null 2>&1
wc -l gpurun_out/ncu_bytes_*.csv
