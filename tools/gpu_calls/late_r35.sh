mkdir -p gpurun_out
python tools/ktimes.py B > gpurun_out/late35_kt.jsonl 2>&1
CURAST_PROVE=0 python tools/ktimes.py B >> gpurun_out/late35_kt.jsonl 2>&1
