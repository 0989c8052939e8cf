mkdir -p gpurun_out
for c in B D C; do python tools/s1_ab.py $c default:CURAST_LIB=tools/ab/base.so 15 2 >> gpurun_out/late65_ab.jsonl 2>&1; done
