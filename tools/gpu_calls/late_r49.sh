mkdir -p gpurun_out
python tools/s1_ab.py C default:CURAST_LIB=tools/ab/base.so 20 3 > gpurun_out/late49_ab.jsonl 2>&1
