mkdir -p gpurun_out
for c in B A C; do python tools/s1_ab.py $c default:CURAST_LIB=tools/ab/r1.so:CURAST_LIB=tools/ab/c1.so:CURAST_LIB=tools/ab/rc1.so 15 2 >> gpurun_out/late60_ab.jsonl 2>&1; done
