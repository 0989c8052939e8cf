mkdir -p gpurun_out
for c in B D C; do python tools/s1_ab.py $c default:CURAST_LIB=tools/ab/x6.so:CURAST_LIB=tools/ab/x7.so 10 2 >> gpurun_out/late78_ab.jsonl 2>&1; done
