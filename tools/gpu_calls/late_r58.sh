mkdir -p gpurun_out
python tools/s1_ab.py Bq default:CURAST_LIB=tools/ab/wp0.so 15 3 > gpurun_out/late58_ab.jsonl 2>&1
