#!/bin/bash
# Round-2 final evidence at HEAD: tools/round2_final.sh (tests, smoke, bench lines, ncu
# launch lists, K6 --set full) plus the N>1 defaults priced on one GPU (one-rank NCCL
# group, reduce-scatter hook, CUDA-graph replay) at the per-rank shapes, and memcheck of
# a small fused step.
export FINAL_DIR=${FINAL_DIR:-r2s3}
bash tools/round2_final.sh
D=gpurun_out/$FINAL_DIR
for t in 2048 4096 8192; do
  timeout -s KILL 300 python bench.py --tokens $t --no-cpu --no-parity --force-dist --graph \
    > $D/proxy_c4_${t}_dist_graph.json 2>/dev/null
done
python tools/primitive_sweep.py > $D/c2_primitive_sweep.jsonl 2>/dev/null
timeout -s KILL 900 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_layer.py -q -x \
  -p no:cacheprovider > $D/memcheck.txt 2>&1; echo rc=$? >> $D/memcheck.txt
tail -3 $D/memcheck.txt
