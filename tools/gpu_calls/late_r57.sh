mkdir -p gpurun_out
python tools/s1_ab.py B default:CURAST_LIB=tools/ab/probe1.so:CURAST_LIB=tools/ab/probe2.so 15 3 > gpurun_out/late57_ab.jsonl 2>&1
