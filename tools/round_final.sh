#!/bin/bash
# End-of-round measurement on one box: tests, smoke, bench lines for every config,
# the reference arm, the ncu launch list + DRAM bytes of one C4 and C3 step.
mkdir -p gpurun_out/final
PYTHONUNBUFFERED=1 timeout -s KILL 400 python -m pytest tests -m gpu -q --timeout 200 -p no:cacheprovider > gpurun_out/final/pytest.txt 2>&1
tail -2 gpurun_out/final/pytest.txt
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.txt 2>&1; tail -2 gpurun_out/final/smoke.txt
timeout -s KILL 400 python bench.py > gpurun_out/final/bench_c4.json 2> gpurun_out/final/bench_c4.err
for c in c3 c5 c1 c4gqa; do
  timeout -s KILL 400 python bench.py --config $c > gpurun_out/final/bench_$c.json 2> gpurun_out/final/bench_$c.err
done
timeout -s KILL 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/bench_reference.json 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in c4 c3; do
  timeout -s KILL 600 ncu --metrics $M --clock-control none --nvtx --nvtx-include "measure/" --csv \
    --log-file gpurun_out/final/ncu_dram_$c.csv python bench.py --config $c --ncu --steps 1 --warmup 1 > /dev/null 2>&1
  cp gpurun_out/launch_tags_$c.json gpurun_out/final/ 2>/dev/null
done
ls gpurun_out/final
