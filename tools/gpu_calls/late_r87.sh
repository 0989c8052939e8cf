mkdir -p gpurun_out
for c in B E200; do python tools/s1_ab.py $c default:CURAST_LIB=tools/ab/k2.so:CURAST_LIB=tools/ab/k4.so 10 2 >> gpurun_out/late87_ab.jsonl 2>&1; done
