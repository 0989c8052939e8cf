mkdir -p gpurun_out
python tools/s1_ab.py C default:CURAST_LIB=tools/ab/base.so 20 2 > gpurun_out/late46_ab.jsonl 2>&1
python tools/s1_ab.py B default:CURAST_LIB=tools/ab/base.so 20 2 >> gpurun_out/late46_ab.jsonl 2>&1
python tools/s1_ab.py A default:CURAST_LIB=tools/ab/base.so 20 2 >> gpurun_out/late46_ab.jsonl 2>&1
