mkdir -p gpurun_out
python tools/s1_ab.py B default:CURAST_LIB=tools/ab/qcs.so:CURAST_LIB=tools/ab/ics.so:CURAST_LIB=tools/ab/bcs.so 15 2 > gpurun_out/late66_ab.jsonl 2>&1
python tools/s1_ab.py E200 default:CURAST_LIB=tools/ab/qcs.so:CURAST_LIB=tools/ab/ics.so:CURAST_LIB=tools/ab/bcs.so 8 1 >> gpurun_out/late66_ab.jsonl 2>&1
