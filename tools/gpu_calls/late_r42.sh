mkdir -p gpurun_out
python tools/s1_ab.py B default:CURAST_SPEC=0:CURAST_LIB=tools/ab/nopf.so 20 3 > gpurun_out/late42_ab_B.jsonl 2>&1
CURAST_SPEC=4 python tools/ktimes.py B 2>/dev/null | grep "^{" >> gpurun_out/late42_kt.jsonl
