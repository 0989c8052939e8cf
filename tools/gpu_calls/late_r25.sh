mkdir -p gpurun_out
python tools/s1_ab.py B default:CURAST_LIB=tools/ab/pad32.so:CURAST_LIB=tools/ab/pad96.so 20 2 > gpurun_out/r25_ab_B.jsonl 2>&1
