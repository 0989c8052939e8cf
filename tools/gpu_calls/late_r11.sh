mkdir -p gpurun_out
python tools/s1_ab.py B default:CURAST_LIB=tools/ab/xpf0.so 20 3 > gpurun_out/r11_ab_B.jsonl 2>&1
python tools/s1_ab.py C default:CURAST_LIB=tools/ab/xpf0.so 20 2 > gpurun_out/r11_ab_C.jsonl 2>&1
