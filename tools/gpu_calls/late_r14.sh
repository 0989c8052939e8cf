mkdir -p gpurun_out
python tools/s1_ab.py B default:CURAST_LIB=tools/ab/base.so:CURAST_LIB=tools/ab/w0.so 20 3 > gpurun_out/r14_ab_B.jsonl 2>&1
python tools/s1_ab.py C default:CURAST_LIB=tools/ab/base.so 15 2 > gpurun_out/r14_ab_C.jsonl 2>&1
python tools/s1_ab.py D default:CURAST_LIB=tools/ab/base.so 10 2 > gpurun_out/r14_ab_D.jsonl 2>&1
