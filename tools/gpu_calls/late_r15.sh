mkdir -p gpurun_out
python tools/s1_ab.py B default:CURAST_LIB=tools/ab/l1.so 20 3 > gpurun_out/r15_ab_B.jsonl 2>&1
