mkdir -p gpurun_out/${PROF_DIR:-r1b}
for s in ${PROF_IDS:-1 6 8 9}; do
timeout -s KILL 400 ncu --set full --clock-control none --import-source on -k regex:coda_gemm_fast -s $s -c 1 -o gpurun_out/${PROF_DIR:-r1b}/prof_s$s python bench.py --ncu --steps 1 --warmup 1 > gpurun_out/${PROF_DIR:-r1b}/prof_s$s.log 2>&1
tail -3 gpurun_out/${PROF_DIR:-r1b}/prof_s$s.log
done
ls -la gpurun_out/${PROF_DIR:-r1b}
