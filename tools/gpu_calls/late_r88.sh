mkdir -p gpurun_out
for c in D Dq C; do python tools/s1_ab.py $c default:CURAST_LIB=tools/ab/base.so 8 2 >> gpurun_out/late88_ab.jsonl 2>&1; done
