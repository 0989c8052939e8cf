mkdir -p gpurun_out
for c in B E200 D C; do python tools/s1_ab.py $c default:CURAST_LIB=tools/ab/base.so 10 2 >> gpurun_out/late70_ab.jsonl 2>&1; done
