mkdir -p gpurun_out
python tools/ktimes.py B 2>/dev/null | grep "^{" > gpurun_out/late39_kt.jsonl
CURAST_SPEC=0 python tools/ktimes.py B 2>/dev/null | grep "^{" >> gpurun_out/late39_kt.jsonl
python tools/s1_ab.py B default:CURAST_SPEC=0 20 2 > gpurun_out/late39_ab_B.jsonl 2>&1
