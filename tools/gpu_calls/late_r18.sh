mkdir -p gpurun_out
python tools/s1_ab.py B CURAST_PIPE=0:CURAST_PIPE=2:CURAST_PIPE=3:CURAST_PIPE=4 20 3 > gpurun_out/r18_ab_B.jsonl 2>&1
