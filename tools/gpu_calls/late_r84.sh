mkdir -p gpurun_out
for c in B E200; do python tools/s1_ab.py $c default:CURAST_LIB=tools/ab/c4k.so:CURAST_LIB=tools/ab/c8k.so 10 2 >> gpurun_out/late84_ab.jsonl 2>&1; done
