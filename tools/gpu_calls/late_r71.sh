mkdir -p gpurun_out
for c in B E200 C A; do python tools/s1_ab.py $c default:CURAST_LIB=tools/ab/ccs.so 10 2 >> gpurun_out/late71_ab.jsonl 2>&1; done
