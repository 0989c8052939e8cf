mkdir -p gpurun_out
for c in Bq Dq; do python tools/s1_ab.py $c default:CURAST_LIB=tools/ab/u16el.so:CURAST_LIB=tools/ab/pkcs.so:CURAST_LIB=tools/ab/both.so 8 2 >> gpurun_out/late72_ab.jsonl 2>&1; done
