mkdir -p gpurun_out
for c in B E200 C A; do python tools/s1_ab.py $c CURAST_LIB=tools/ab/cur.so:CURAST_LIB=tools/ab/m7.so:CURAST_LIB=tools/ab/m6.so 10 2 >> gpurun_out/late98_ab.jsonl 2>&1; done
