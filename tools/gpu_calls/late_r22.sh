mkdir -p gpurun_out
python tools/s1_ab.py B CURAST_FUSE=0:CURAST_FUSE=4:CURAST_FUSE=3:CURAST_FUSE=2 20 2 > gpurun_out/r22_ab_B.jsonl 2>&1
python tools/s1_ab.py C CURAST_FUSE=0:CURAST_FUSE=4:CURAST_FUSE=3 10 1 > gpurun_out/r22_ab_C.jsonl 2>&1
python tools/s1_ab.py A CURAST_FUSE=0:CURAST_FUSE=4:CURAST_FUSE=3 10 1 > gpurun_out/r22_ab_A.jsonl 2>&1
