mkdir -p gpurun_out
python tools/s1_ab.py B default:CURAST_LIB=tools/ab/m5.so 15 2 > gpurun_out/late62_ab.jsonl 2>&1
