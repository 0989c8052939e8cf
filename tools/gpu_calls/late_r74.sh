mkdir -p gpurun_out
for c in B E200 C; do python tools/s1_ab.py $c default:CURAST_LIB=tools/ab/rp.so 10 2 >> gpurun_out/late74_ab.jsonl 2>&1; done
