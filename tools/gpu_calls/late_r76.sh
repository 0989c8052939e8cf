mkdir -p gpurun_out
for c in B E200; do python tools/s1_ab.py $c default:CURAST_LIB=tools/ab/cv0.so:CURAST_LIB=tools/ab/cv25.so 10 2 >> gpurun_out/late76_ab.jsonl 2>&1; done
