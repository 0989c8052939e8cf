mkdir -p gpurun_out
for c in A4 C A D; do python tools/s1_ab.py $c default:CURAST_LIB=tools/ab/w16.so 10 2 >> gpurun_out/late50_ab.jsonl 2>&1; done
