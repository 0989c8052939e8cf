mkdir -p gpurun_out
python tools/s1_ab.py B default:CURAST_LIB=tools/ab/m3.so:CURAST_LIB=tools/ab/m2.so 15 2 > gpurun_out/late61_ab.jsonl 2>&1
