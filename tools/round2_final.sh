#!/bin/bash
# Round-2 measurement on one box: GPU tests, smoke, bench lines (C4 default + fold variant,
# C3, C5, C1, C4-GQA, the reference arm, per-rank shape proxies), ncu launch lists with DRAM
# bytes of one C4 and C3 step, and a --set full capture of the roofline kernel (K6).
D=gpurun_out/${FINAL_DIR:-final2}
mkdir -p $D
PYTHONUNBUFFERED=1 timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > $D/pytest.txt 2>&1
tail -2 $D/pytest.txt
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1; tail -2 $D/smoke.txt
timeout -s KILL 400 python bench.py > $D/bench_c4.json 2> $D/bench_c4.err
timeout -s KILL 400 python bench.py --fold-gamma --no-cpu > $D/bench_c4_fold.json 2> $D/bench_c4_fold.err
for c in c3 c5 c1 c4gqa; do
  timeout -s KILL 400 python bench.py --config $c > $D/bench_$c.json 2> $D/bench_$c.err
done
for t in 2048 4096 8192; do
  timeout -s KILL 300 python bench.py --tokens $t --no-cpu --no-parity > $D/proxy_c4_$t.json 2>/dev/null
done
timeout -s KILL 400 python bench.py --impl reference --steps 3 --warmup 3 > $D/bench_reference.json 2>&1
M=gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum
for c in c4 c3; do
  timeout -s KILL 600 ncu --metrics $M --clock-control none --nvtx --nvtx-include "measure/" --csv \
    --log-file $D/ncu_launches_$c.csv python bench.py --config $c --ncu --steps 1 --warmup 1 > /dev/null 2>&1
  cp gpurun_out/launch_tags_$c.json $D/ 2>/dev/null
done
PROF_DIR=${FINAL_DIR:-final2} PROF_IDS="1" bash tools/prof_nvtx.sh > /dev/null 2>&1
ls $D
