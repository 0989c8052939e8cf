mkdir -p gpurun_out
python tools/ktimes.py B > gpurun_out/late36_kt.jsonl 2>&1
CURAST_PROVE=0 python tools/ktimes.py B >> gpurun_out/late36_kt.jsonl 2>&1
python tools/s1_ab.py B default:CURAST_PROVE=0 20 2 > gpurun_out/late36_ab_B.jsonl 2>&1
python tools/s1_ab.py C default:CURAST_PROVE=0 10 1 > gpurun_out/late36_ab_C.jsonl 2>&1
