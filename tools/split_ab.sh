python tools/gemm_bench.py --shape 4096,4096,4096 --shape 2048,28672,4096 --shape 16384,14336,4096,0,1 --shape 8192,2048,2048 --variant split_min_k=8192,split_piece_kb=4 --variant split_min_k=4096,split_piece_kb=32 --variant split_min_k=4096,split_piece_kb=16 --variant split_min_k=2048,split_piece_kb=32 > gpurun_out/gb_split2.txt 2>&1
V="--variant split_min_k=8192,split_piece_kb=4 --variant split_min_k=4096,split_piece_kb=32 --variant split_min_k=4096,split_piece_kb=16"
python tools/ab_inproc.py --config c4 --rounds 10 $V > gpurun_out/ab2_c4.json 2>&1
python tools/ab_inproc.py --config c4 --tokens 2048 --rounds 16 $V > gpurun_out/ab2_c4_2048.json 2>&1
python tools/ab_inproc.py --config c3 --rounds 16 $V > gpurun_out/ab2_c3.json 2>&1
