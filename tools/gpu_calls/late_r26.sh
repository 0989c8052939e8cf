mkdir -p gpurun_out
python tools/s1_ab.py B default:CURAST_LIB=tools/ab/px0.so:CURAST_LIB=tools/ab/base.so 20 3 > gpurun_out/r26_ab_B.jsonl 2>&1
python tools/s1_ab.py C default:CURAST_LIB=tools/ab/base.so 10 2 > gpurun_out/r26_ab_C.jsonl 2>&1
python tools/s1_ab.py A default:CURAST_LIB=tools/ab/base.so 10 2 > gpurun_out/r26_ab_A.jsonl 2>&1
