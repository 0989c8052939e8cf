mkdir -p gpurun_out
for c in B D C A; do python tools/s1_ab.py $c default:CURAST_LIB=tools/ab/base.so 10 2 >> gpurun_out/late79_ab.jsonl 2>&1; done
