mkdir -p gpurun_out
python tools/s1_ab.py C default:CURAST_LIB=tools/ab/base.so 20 2 > gpurun_out/late32_ab_C.jsonl 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_stage2" -s 2 -c 1 -o gpurun_out/late32_C python tools/frame_once.py C 3 > gpurun_out/late32_ncu.log 2>&1
