mkdir -p gpurun_out
for c in B E200 C D A; do python tools/s1_ab.py $c default:CURAST_LIB=tools/ab/xcs.so:CURAST_LIB=tools/ab/nocs.so 12 2 >> gpurun_out/late67_ab.jsonl 2>&1; done
